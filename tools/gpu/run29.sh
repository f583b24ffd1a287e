FASTPFP_LIB=build/var_atmem/libfastpfp.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "int8_ozaki_error_bound" 2>&1 | tail -3
FASTPFP_LIB=build/var_atmem/libfastpfp.so timeout 300 python tools/prec_time.py c5 3 2>&1 | tail -1
