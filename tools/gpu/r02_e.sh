timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/g5_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/g5_tests.log
timeout 300 python bench.py --workload c4 --steps 200 --warmup 3 > gpurun_out/g5_c4.json 2>&1; echo "c4 rc=$?"; tail -2 gpurun_out/g5_c4.json | cut -c1-300
