timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/g17_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g17_tests.log
FASTPFP_LIB=varlib/var_projprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c5 2 2>&1 | grep -E "proj-prof|ok" | head -6
