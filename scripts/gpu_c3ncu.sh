#!/bin/bash
# ncu --set full of one prepared-W C3 GEMM launch per kernel variant (flags: 0 = default, 16384 = k_modgemm_tcs)
mkdir -p gpurun_out
for f in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_tc -s 6 -c 1 -o gpurun_out/prof_c3_$f python scripts/gemm_probe.py 1024 256 --tc-only --prepared --flags=$f > gpurun_out/ncu_c3_$f.log 2>&1
done
