timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/g21_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g21_tests.log
FASTPFP_LIB=varlib/var_ssprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c4 20 2>&1 | grep -E "ss-prof|ok" | head -5
for i in 1 2; do timeout 300 python bench.py --workload c4 --steps 400 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['value'])"; done
