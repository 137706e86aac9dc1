#!/bin/bash
# A/B of the single-party MAC sigma's ALU/fma split (SPDZ_SIGMA1_ALU_SHIFTS builds): the bench's
# per-party block (sigma<1> GB/s inside the per-party step, one stream and chunked), interleaved twice
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" variants/v_s1_7/libspdz_b200.so variants/v_s1_3/libspdz_b200.so variants/v_s1_5/libspdz_b200.so; do
  echo -n "lib=$v " >> gpurun_out/s1ab.log
  SPDZ_B200_LIB=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-linear --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['per_party']; print(round(d['ms_per_step'],4), d['roofline']['all_kernels_gbs']['sigma'], round(p['ms_per_step'],4), p['kernels_gbs']['sigma'], round(p['chunked']['ms_per_step'],4))" >> gpurun_out/s1ab.log 2>&1
done
done
