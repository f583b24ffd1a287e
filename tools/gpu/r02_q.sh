# on-chip tagged exchange (final form) parity + c2/c3 timing; c4 with/without warp reconvergence
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py -x -q > gpurun_out/g28_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g28_tests.log
timeout 300 python - <<'PY'
import sys, json; sys.path.insert(0, ".")
import bench
for c in ("c2", "c3", "c1"):
    r = bench.secondary_pair(c)
    print(c, json.dumps({k: r[k] for k in ("value", "solve_ms", "ms_per_sweep", "total_sweeps", "proj_kernel")}))
PY
for v in "" varlib/var_sssw/libfastpfp.so "" varlib/var_sssw/libfastpfp.so; do
FASTPFP_LIB=$v timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "
import json,sys,os; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
