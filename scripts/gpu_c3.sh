#!/bin/bash
# C3 GEMM A/B: GEMM parity tests, then the probe for the default path and each diagnostic flag set given
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_surface.py -q -m gpu -x -k "linear or prepared or batched or gemm" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
for f in 0 "$@"; do
  echo "== flags $f" >> gpurun_out/c3.log
  timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --prepared --flags=$f >> gpurun_out/c3.log 2>&1
done
