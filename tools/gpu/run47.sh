timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r47_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r47_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r47_bench.json 2> gpurun_out/r47_bench.err; echo "bench rc=$?"
