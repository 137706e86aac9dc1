#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/step_modes_probe.py > gpurun_out/fuse2.log 2>&1
SPDZ_NO_MASK_FUSION=1 timeout 300 python scripts/step_modes_probe.py > gpurun_out/fuse2_off.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
