#!/bin/bash
# C3 GEMM iteration: kernel tests, variant timings, timelines, one ncu capture of k_modgemm_tcs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "linear or prepared or batched" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --variants --timeline --tl-flags=0 > gpurun_out/gemm_variants.log 2>&1
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --timeline --tl-flags=0 --tl-prepared >> gpurun_out/gemm_variants.log 2>&1
timeout 300 python scripts/gemm_probe.py 8192 1024 --tc-only >> gpurun_out/gemm_variants.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_tcs -s 3 -c 1 -o gpurun_out/prof_gemm_tcs python scripts/gemm_probe.py 1024 256 --tc-only > gpurun_out/ncu_gemm_tcs.log 2>&1
