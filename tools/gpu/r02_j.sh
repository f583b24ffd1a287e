FASTPFP_LIB=varlib/var_projprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c5 2 2>&1 | grep -E "proj-prof|ok" | head -6
timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/g18_bench.json 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/g18_bench.json').read().splitlines() if l.startswith('{')][-1])
r=d['roofline']; print(d['value'], d['ms_per_step'], 'gemm', r['ms_per_launch'], 'proj', r['secondary']['ms_per_launch'], r['secondary']['frac'], d['clocks'])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pg.py tests/test_gpu_api.py -x -q > gpurun_out/g18_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g18_tests.log
