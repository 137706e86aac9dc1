#!/bin/bash
# A/B of the MAC-sigma pipe balance (SPDZ_SIGMA_ALU_SHIFTS / SPDZ_SIGMA_ALU_FIVE builds): single-party
# ceiling, and the bench step (co-located sigma<2> and the per-party sigma<1> GB/s)
mkdir -p gpurun_out
for v in "" variants/v_s7f/libspdz_b200.so variants/v_s3f/libspdz_b200.so variants/v_s5f/libspdz_b200.so variants/v_s1f/libspdz_b200.so; do
  SPDZ_B200_LIB=$v timeout 300 python scripts/sigma_ceiling.py >> gpurun_out/sigma_ab.jsonl 2>>gpurun_out/sigma_ab.err
done
for v in "" variants/v_s7f/libspdz_b200.so variants/v_s3f/libspdz_b200.so; do
  echo "lib=$v" >> gpurun_out/sigma_bench.log
  SPDZ_B200_LIB=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-linear --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['all_kernels_gbs'], d['per_party']['ms_per_step'], d['per_party']['kernels_gbs'])" >> gpurun_out/sigma_bench.log 2>&1
done
