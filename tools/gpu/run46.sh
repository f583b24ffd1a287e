timeout 300 python tools/proj_time.py
timeout 600 python tools/prec_time.py c5 3 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "streaming or config5 or sweeps_vs or dist" 2>&1 | tail -2
