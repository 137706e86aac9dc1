#!/bin/bash
# C3 GEMM: parity tests, variants side by side, timelines of the default and the previous kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_surface.py -q -m gpu -x -k "linear or prepared or batched or gemm" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --variants > gpurun_out/c3_variants.log 2>&1
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --timeline --tl-prepared --tl-flags=0,16384 > gpurun_out/c3_timeline.log 2>&1
