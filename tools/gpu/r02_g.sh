timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/g12_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g12_tests.log
FASTPFP_LIB=varlib/var_ssprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c4 20 2>&1 | grep -E "ss-prof|ok" | head -5
timeout 300 python bench.py --workload c4 --steps 200 --warmup 3 > gpurun_out/g12_c4.json 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/g12_c4.json | cut -c1-200
