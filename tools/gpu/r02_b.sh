# discretize v2 + sharded-path changes + new bench line
timeout 900 python -m pytest tests/test_gpu_parity.py -k "greedy" tests/test_gpu_dist.py tests/test_gpu_api.py tests/test_gpu_batched.py -x -q > gpurun_out/g2_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g2_tests.log
timeout 300 python tools/ncu_driver.py discretize 16384 > gpurun_out/g2_disc.log 2>&1; echo "disc rc=$?"; tail -4 gpurun_out/g2_disc.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g2_bench.err
timeout 600 python bench.py --workload c4 --steps 200 --warmup 3 > gpurun_out/g2_bench_c4.json 2> gpurun_out/g2_bench_c4.err; echo "c4 rc=$?"
