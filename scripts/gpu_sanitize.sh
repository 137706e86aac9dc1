#!/bin/bash
# compute-sanitizer over the GPU suite on the current kernels:
#  memcheck: every GPU test except the full-size headline ones (2^24 / 2^28 lanes) and the
#            multi-process / network ones (child processes);
#  racecheck + synccheck: the kernels with shared-memory / cluster protocols (split-K cluster GEMM,
#            tcgen05 GEMMs, co-located matrix combine and linear mask, MAC sigma, node streams).
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='not 2p24 and not 2p28 and not multiprocess and not one_party_per_process and not net'
timeout 3000 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_runtime.py tests/test_gpu_surface.py tests/test_gpu_scheduler.py tests/test_gpu_headline.py -q -m gpu -k "$SEL" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log
SEL2='linear or prepared or gemm or batched or matrix or sigma'
timeout 1500 $CS --tool racecheck --racecheck-report all --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "$SEL2" > gpurun_out/racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "$SEL2" > gpurun_out/synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/synccheck.log
timeout 900 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_scheduler.py tests/test_gpu_runtime.py -q -m gpu -k "node_streams or linear" > gpurun_out/racecheck_runtime.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck_runtime.log
