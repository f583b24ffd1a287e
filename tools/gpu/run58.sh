ncu --set full --import-source on --clock-control none -k regex:gemm_i8 -s 2 -c 1 -o gpurun_out/i8_norm python tools/prec_time.py c5 3 > gpurun_out/ncu58a.log 2>&1
FASTPFP_LIB=varlib/dp.so ncu --set full --import-source on --clock-control none -k regex:gemm_i8 -s 2 -c 1 -o gpurun_out/i8_dp python tools/prec_time.py c5 3 > gpurun_out/ncu58b.log 2>&1
