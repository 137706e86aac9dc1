#!/bin/bash
# A/B of the software-pipelined two-party MAC sigma (SPDZ_SIGMA2_PIPE builds): C4 probe and the chain step
mkdir -p gpurun_out
for v in "" variants/v_pipe2/libspdz_b200.so variants/v_pipe3/libspdz_b200.so; do
  echo "lib=$v" >> gpurun_out/sigma_pipe.log
  SPDZ_B200_LIB=$v timeout 200 python scripts/linear_probe.py >> gpurun_out/sigma_pipe.log 2>&1
  SPDZ_B200_LIB=$v timeout 300 python scripts/step_modes_probe.py >> gpurun_out/sigma_pipe.log 2>&1
done
SPDZ_B200_LIB=variants/v_pipe2/libspdz_b200.so timeout 600 python -m pytest tests -q -m gpu -x -k "sigma or mac or chain or linear" > gpurun_out/pt_pipe2.log 2>&1
