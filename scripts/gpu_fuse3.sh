#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for k in mixed heavy; do
  echo "== $k on" >> gpurun_out/fuse3.log; timeout 300 python scripts/step_modes_probe.py 16777216 $k >> gpurun_out/fuse3.log 2>&1
  echo "== $k off" >> gpurun_out/fuse3.log; SPDZ_NO_MASK_FUSION=1 timeout 300 python scripts/step_modes_probe.py 16777216 $k >> gpurun_out/fuse3.log 2>&1
done
