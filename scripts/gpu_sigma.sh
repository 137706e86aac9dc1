#!/bin/bash
# single-party MAC sigma: L2 ceiling vs HBM, and one source-level ncu capture (stall reasons per SASS line)
mkdir -p gpurun_out
timeout 300 python scripts/sigma_ceiling.py > gpurun_out/sigma_ceiling.jsonl 2>&1
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --section Occupancy --section ComputeWorkloadAnalysis --warp-sampling-interval 2 --clock-control none --import-source on -k regex:k_mac_sigma -s 6 -c 1 -o gpurun_out/prof_sigma1 python scripts/sigma_ceiling.py > gpurun_out/ncu_sigma1.log 2>&1
