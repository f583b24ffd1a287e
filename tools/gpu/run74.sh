M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum.per_second,dram__bytes_write.sum.per_second
ncu --metrics $M --clock-control none -k regex:proj_kernel -s 1 -c 2 --csv python tools/prec_time.py c5 3 > gpurun_out/ncu74_new.csv 2>&1
FASTPFP_LIB=varlib/projold.so ncu --metrics $M --clock-control none -k regex:proj_kernel -s 1 -c 2 --csv python tools/prec_time.py c5 3 > gpurun_out/ncu74_old.csv 2>&1
