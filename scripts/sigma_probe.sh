#!/bin/bash
# A/B of MAC-sigma kernel builds: single-party sigma (compute ceiling / HBM) and the 2-party step.
mkdir -p gpurun_out
for v in "" build/v_lock/libspdz_b200.so; do
  SPDZ_B200_LIB=$v timeout 300 python scripts/sigma_ceiling.py >> gpurun_out/sigma_probe.jsonl 2>>gpurun_out/sigma_probe.err
done
SPDZ_B200_LIB=build/v_lock/libspdz_b200.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "sigma or coefficient" > gpurun_out/sigma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sigma_tests.log
