#!/bin/bash
# e2e chunking sweep (host-streamed, one deferred MAC check, pinned inputs)
mkdir -p gpurun_out
for w in "" "1,1,1,1,1,1,1,1,1,1,1,1" "2,2,2,2,2,2,2,1,1" "4,4,4,4,4,4,4,2,1,1" "1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1" "3,3,3,3,3,3,3,2,1"; do
  echo "weights=$w" >> gpurun_out/e2e_sweep.log
  if [ -z "$w" ]; then A=""; else A="--e2e-weights $w"; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-linear --no-cpu-baseline --no-per-party $A 2>&1 >/dev/null | grep "e2e joint MAC check, pinned" >> gpurun_out/e2e_sweep.log
done
