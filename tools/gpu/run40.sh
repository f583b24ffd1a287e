timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "int8_ozaki_error_bound or blocked" 2>&1 | tail -3
timeout 600 python tools/prec_time.py c5 3 | tail -1
