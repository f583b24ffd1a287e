timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/g4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g4_tests.log
timeout 300 python bench.py --workload c4 --steps 200 --warmup 3 > gpurun_out/g4_c4.json 2>&1; echo "c4 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/g4_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
FASTPFP_LIB=varlib/var_ssprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c4 20 2>&1 | grep -E "ss-prof|ok" | head -3
