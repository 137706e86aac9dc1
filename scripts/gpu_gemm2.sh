#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_modgemm_tcs -s 3 -c 1 -o gpurun_out/prof_gemm_tcs_src python scripts/gemm_probe.py 1024 256 --tc-only --flags=8192 > gpurun_out/ncu_gemm_tcs.log 2>&1
