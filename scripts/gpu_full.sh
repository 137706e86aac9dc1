#!/bin/bash
# Full evidence capture on one B200: GPU tests, smoke, bench (+ the reference arm on the same
# workload), ncu launch list of the bench command, ncu --set full of the dominant kernels, the
# reference's kernel microbenchmarks, the BASELINE config sweep, C4 / C3 probes.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "$SKIP_REF" ]; then
  s=$(date +%s); timeout 1500 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/bench_ref.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-linear --no-per-party > gpurun_out/ncu_launch.log 2>&1
NB="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-linear --no-per-party"
NC="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
# the timed step's first combine (the next multiply's mask fused), its mask and its MAC sigma
timeout 600 $NC -k regex:OpCombine2 -s 4 -c 1 -o gpurun_out/prof_combine $NB > gpurun_out/ncu_combine.log 2>&1
timeout 600 $NC -k regex:OpMask2 -s 1 -c 1 -o gpurun_out/prof_mask $NB > gpurun_out/ncu_mask.log 2>&1
timeout 600 $NC -k regex:k_mac_sigma -s 1 -c 1 -o gpurun_out/prof_sigma $NB > gpurun_out/ncu_sigma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_matrix_combine2 -s 2 -c 1 -o gpurun_out/prof_matrix_combine2 python scripts/linear_probe.py > gpurun_out/ncu_mc2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_tcs -s 6 -c 1 -o gpurun_out/prof_gemm_tcs python scripts/gemm_probe.py 1024 256 --tc-only --prepared > gpurun_out/ncu_gemm.log 2>&1
timeout 600 python scripts/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
timeout 300 python scripts/linear_probe.py > gpurun_out/linear_probe.log 2>&1
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --variants > gpurun_out/gemm_variants.log 2>&1
timeout 1800 python bench_configs.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep.log
ls -la gpurun_out
