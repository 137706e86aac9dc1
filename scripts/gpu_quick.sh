#!/bin/bash
# Quick gpurun call: GPU tests, bench, quick sweep (+ optional ncu of a kernel regex in $NCU_K)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench_configs.py --quick --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep.log
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$NCU_K" -s ${NCU_S:-2} -c 1 -o gpurun_out/prof_${NCU_TAG:-k} ${NCU_CMD:-python bench_configs.py --quick --no-ref --out /tmp/s.json} > gpurun_out/ncu_${NCU_TAG:-k}.log 2>&1
fi
