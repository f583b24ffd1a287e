# fp32 warp max via redux.sync (CREDUX) vs the shuffle butterfly: parity + c4/c2 timing
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -x -q > gpurun_out/g29_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g29_tests.log
for v in "" varlib/var_noredux/libfastpfp.so "" varlib/var_noredux/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
timeout 300 python - <<'PY'
import sys, os, json; sys.path.insert(0, ".")
import bench
r = bench.secondary_pair("c2")
print(os.environ.get("FASTPFP_LIB") or "main", "c2", json.dumps({k: r[k] for k in ("value", "ms_per_sweep")}))
PY
done
