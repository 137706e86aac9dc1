#!/bin/bash
# Evidence run: GPU tests, smoke, bench (+reference arm), full sweep, ncu launch list of the
# bench command, ncu --set full of the dominant kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1200 python bench_configs.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:OpCombine -s 4 -c 1 -o gpurun_out/prof_combine python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/ncu_combine.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_sigma -s 2 -c 1 -o gpurun_out/prof_sigma python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/ncu_sigma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:OpMask -s 4 -c 1 -o gpurun_out/prof_mask python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-chunks 1 > gpurun_out/ncu_mask.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_modgemm_tc -s 1 -c 1 -o gpurun_out/prof_gemm_tc python scripts/gemm_probe.py 8192 1024 > gpurun_out/ncu_gemm.log 2>&1

timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_matrix_combine2 -s 2 -c 1 -o gpurun_out/prof_matrix_combine2 python scripts/linear_probe.py > gpurun_out/ncu_mc2.log 2>&1
timeout 300 python scripts/streamed_timeline.py 8 > gpurun_out/timeline.log 2>&1
timeout 600 python scripts/kernel_bench.py > gpurun_out/kernel_bench.json 2> gpurun_out/kernel_bench.err
timeout 300 python scripts/linear_probe.py > gpurun_out/linear_probe.log 2>&1
for s in "1024 256" "8192 1024"; do timeout 300 python scripts/gemm_probe.py $s --tc-only --diag --prepared; done > gpurun_out/gemm_diag.log 2>&1

ls -la gpurun_out
