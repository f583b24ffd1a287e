FASTPFP_LIB=build/var_ssprof/libfastpfp.so timeout 300 python tools/c4_split.py 2>&1 | grep ss-prof | head -2
timeout 300 python tools/c4_split.py
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -2
