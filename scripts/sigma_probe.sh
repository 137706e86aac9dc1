#!/bin/bash
# A/B of MAC-sigma kernel builds: compute ceiling (L2-resident) vs HBM stream, and in the heavy-chain step.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "sigma or coefficient" > gpurun_out/sigma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sigma_tests.log
for v in "" build/v_minb4/libspdz_b200.so build/v_minb6/libspdz_b200.so; do
  SPDZ_B200_LIB=$v timeout 300 python scripts/sigma_ceiling.py >> gpurun_out/sigma_probe.jsonl 2>>gpurun_out/sigma_probe.err
  SPDZ_B200_LIB=$v timeout 300 python scripts/reduction_probe.py >> gpurun_out/sigma_probe.jsonl 2>>gpurun_out/sigma_probe.err
done
