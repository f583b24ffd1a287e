set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r1_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench.log 2>gpurun_out/r1_bench.err; echo "bench rc=$?"
cat gpurun_out/r1_bench.log
