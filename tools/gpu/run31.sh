timeout 300 python tools/c4_split.py
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -5
