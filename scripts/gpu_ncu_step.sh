#!/bin/bash
# ncu --set full of the heavy-chain step's kernels (timed step of `bench.py --steps 1 --warmup 1`):
# the first OpCombine2 and OpMask2 launch of the timed step and its MAC sigma.
mkdir -p gpurun_out
NB="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-linear --no-per-party"
NC="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 600 $NC -k regex:OpCombine2 -s 4 -c 1 -o gpurun_out/prof_combine $NB > gpurun_out/ncu_combine.log 2>&1
timeout 600 $NC -k regex:OpMask2 -s 4 -c 1 -o gpurun_out/prof_mask $NB > gpurun_out/ncu_mask.log 2>&1
timeout 600 $NC -k regex:k_mac_sigma -s 1 -c 1 -o gpurun_out/prof_sigma $NB > gpurun_out/ncu_sigma.log 2>&1
