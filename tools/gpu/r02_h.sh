timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_api.py tests/test_gpu_pg.py -x -q > gpurun_out/g13_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g13_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/g13_bench.json 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/g13_bench.json').read().strip().splitlines()[-1])
r=d['roofline']; print(d['value'], d['ms_per_step'], 'gemm', r['ms_per_launch'], r['frac'], 'proj', r['secondary']['ms_per_launch'], r['secondary']['frac'], d['clocks'])
PY
