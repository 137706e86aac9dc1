#!/bin/bash
# tcgen05 GEMM v2 vs v1: parity tests, then timings at the C3 shape and the batched large shapes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "linear_secret_public" -x > gpurun_out/gemm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_tests.log
for shape in "1024 256" "4096 1024" "8192 1024"; do
  for v in "" "--v1"; do
    echo "== $shape $v" >> gpurun_out/gemm_ab.log
    timeout 300 python scripts/gemm_probe.py $shape --tc-only $v >> gpurun_out/gemm_ab.log 2>&1
  done
done
