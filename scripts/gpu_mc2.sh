#!/bin/bash
# C4 combine iteration: linear-layer tests, linear probe, one ncu capture of k_matrix_combine2_flat
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_kernels.py -q -m gpu -x -k "linear or matrix" > gpurun_out/pytest_mc2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mc2.log
timeout 300 python scripts/linear_probe.py > gpurun_out/linear_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_matrix_combine2 -s 2 -c 1 -o gpurun_out/prof_mc2 python scripts/linear_probe.py > gpurun_out/ncu_mc2.log 2>&1
