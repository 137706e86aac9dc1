mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_sigma -s 3 -c 1 -o gpurun_out/prof_sigma_stage python scripts/sigma_ceiling.py > gpurun_out/ncu_sig1.log 2>&1
SPDZ_B200_LIB=build/v_minb5/libspdz_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mac_sigma -s 3 -c 1 -o gpurun_out/prof_sigma_minb5 python scripts/sigma_ceiling.py > gpurun_out/ncu_sig2.log 2>&1
