for f in 1 2 3 4; do FUSE=$f timeout 300 python tools/proj_time.py; done
FUSE=1 FASTPFP_LIB=build/var_minb2/libfastpfp.so timeout 300 python tools/proj_time.py
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streaming or config5 or sweeps_vs" 2>&1 | tail -2
