FASTPFP_LIB=build/var_ssprof/libfastpfp.so timeout 300 python tools/c4_split.py 2>&1 | grep -m1 ss-prof
timeout 300 python tools/c4_split.py
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -2
