timeout 600 python tools/prec_time.py c5 3 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pg.py -x -q -k "int8" 2>&1 | tail -2
