timeout 900 python -m pytest tests/test_gpu_ga.py -x -q > gpurun_out/r2_ga.log 2>&1; echo "ga tests rc=$?"
tail -30 gpurun_out/r2_ga.log
timeout 300 python tools/ga_time.py
