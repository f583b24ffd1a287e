FASTPFP_LIB=build/var_ocprof/libfastpfp.so timeout 300 python tools/c2_probe.py 2>&1 | tail -4
timeout 300 python tools/c2_probe.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config2 or config3 or ragged or dyadic or distance or planted" 2>&1 | tail -3
