timeout 300 python tools/proj_time.py
timeout 600 python tools/prec_time.py c5 3 | tail -1
timeout 300 python tools/c2_probe.py 2>&1 | grep "pk 0"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pg.py -x -q 2>&1 | tail -2
