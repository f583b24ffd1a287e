timeout 300 python tools/prec_time.py c5 3 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_pg.py -x -q -k "int8 or blocked or full_size" 2>&1 | tail -2
