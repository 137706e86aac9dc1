#!/bin/bash
# Round-2 evidence (after the C3 kernel): GPU tests, smoke, bench, reference arm at the full size,
# ncu launch list of the bench command, the reference's kernel microbenchmarks through the host API
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
s=$(date +%s); timeout 1500 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-linear --no-per-party > gpurun_out/ncu_launch.log 2>&1
timeout 600 python scripts/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
ls -la gpurun_out
