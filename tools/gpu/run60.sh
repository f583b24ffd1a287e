for i in 1 2; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/dp.so timeout 300 python tools/prec_time.py c5 3 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_pg.py tests/test_gpu_ga.py -x -q -k "int8 or blocked or full_size" 2>&1 | tail -2
