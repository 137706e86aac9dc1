#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-linear --no-cpu-baseline > gpurun_out/bench_pp.json 2> gpurun_out/bench_pp.err
