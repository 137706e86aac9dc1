#!/bin/bash
# C3 split-K kernel check + probe, box memory, reference arm memory at the full size
mkdir -p gpurun_out
{ free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; cat /sys/fs/cgroup/memory/memory.limit_in_bytes 2>/dev/null; nproc; } > gpurun_out/box_mem.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "linear or prepared or batched" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_probe.py 1024 256 --tc-only --variants > gpurun_out/gemm_variants.log 2>&1
timeout 300 python scripts/gemm_probe.py 8192 1024 --tc-only >> gpurun_out/gemm_variants.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_tcs -s 3 -c 1 -o gpurun_out/prof_gemm_tcs python scripts/gemm_probe.py 1024 256 --tc-only > gpurun_out/ncu_gemm_tcs.log 2>&1
( s=$(date +%s); timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/bench_ref.err ) &
BP=$!
while kill -0 $BP 2>/dev/null; do free -m | awk '/Mem/{print $3, $7}' >> gpurun_out/ref_mem.log; sleep 5; done
ls -la gpurun_out
