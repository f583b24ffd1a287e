FASTPFP_LIB=build/var_ssprof/libfastpfp.so timeout 300 python tools/c4_split.py 2>&1 | grep -m1 ss-prof
timeout 300 python tools/c4_split.py
timeout 600 python tools/prec_time.py c5 3 | tail -1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "batched or config4 or int8 or blocked" 2>&1 | tail -2
