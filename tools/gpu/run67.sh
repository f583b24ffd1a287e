timeout 300 python tools/proj_time.py
for i in 1 2; do timeout 300 python tools/prec_time.py c5 3 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
