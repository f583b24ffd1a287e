timeout 300 python tools/ga_time.py
timeout 900 python -m pytest tests/test_gpu_ga.py -x -q 2>&1 | tail -2
