#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "linear or prepared or batched" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --variants > gpurun_out/gemm_variants.log 2>&1
