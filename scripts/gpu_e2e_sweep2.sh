#!/bin/bash
# e2e chunk weights, interleaved 3 times (host-streamed, one deferred MAC check, pinned inputs)
mkdir -p gpurun_out
for rep in 1 2; do
for w in ${WEIGHTS:-"" "4,4,4,4,4,4,4,3,1" "3,3,3,3,3,3,3,2,1,1" "2,2,2,2,2,2,2,2,1"}; do
  if [ -z "$w" ]; then A=""; else A="--e2e-weights $w"; fi
  r=$(timeout 600 python bench.py --steps 10 --warmup 3 --no-linear --no-cpu-baseline --no-per-party $A 2>&1 >/dev/null | grep "e2e joint MAC check, pinned")
  echo "w=$w $r" >> gpurun_out/e2e_sweep2.log
done
done
