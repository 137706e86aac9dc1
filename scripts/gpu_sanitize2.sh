#!/bin/bash
# compute-sanitizer memcheck / racecheck over the runtime tests after the launch fusions
# (OpCombine2M / OpCombine2A / OpCombineM / OpAddSub2 / OpOpen2, the matrix-combine root opening)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='not 2p24 and not 2p28 and not multiprocess and not one_party_per_process and not net and not fusion'
timeout 2400 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_headline.py tests/test_gpu_scheduler.py -q -m gpu -k "$SEL" > gpurun_out/memcheck2.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck2.log
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_runtime.py -q -m gpu -k "chain or linear or graph" > gpurun_out/racecheck2.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/racecheck2.log
