for v in "" build/var_nobulk/libfastpfp.so build/var_slots4/libfastpfp.so build/var_slots8/libfastpfp.so; do FASTPFP_LIB=$v timeout 300 python tools/proj_time.py; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streaming or config5 or sweeps_vs" 2>&1 | tail -2
