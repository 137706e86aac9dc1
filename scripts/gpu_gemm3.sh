#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --timeline --tl-flags=512,520,64,72 > gpurun_out/gemm_pair.log 2>&1
