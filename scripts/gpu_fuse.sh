#!/bin/bash
# mask-into-combine fusion: GPU tests, then the chain step with fusion off / on / on with two lane groups
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for v in off on u2; do
  echo "== $v" >> gpurun_out/fuse.log
  case $v in
    off) SPDZ_NO_MASK_FUSION=1 timeout 300 python scripts/step_modes_probe.py >> gpurun_out/fuse.log 2>&1 ;;
    on) timeout 300 python scripts/step_modes_probe.py >> gpurun_out/fuse.log 2>&1 ;;
    u2) SPDZ_B200_LIB=variants/v_c2m_u2/libspdz_b200.so timeout 300 python scripts/step_modes_probe.py >> gpurun_out/fuse.log 2>&1 ;;
  esac
done
