M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
ncu --metrics $M --clock-control none -k regex:gemm_i8 -s 2 -c 2 --csv python tools/prec_time.py c5 3 > gpurun_out/ncu57_norm.csv 2>&1
FASTPFP_LIB=varlib/dp.so ncu --metrics $M --clock-control none -k regex:gemm_i8 -s 2 -c 2 --csv python tools/prec_time.py c5 3 > gpurun_out/ncu57_dp.csv 2>&1
