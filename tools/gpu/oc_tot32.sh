# c2/c3 A/B: 8-byte tile totals and deltas too (FPFP_OC_TOT32) vs main
FASTPFP_LIB=varlib/var_tot32/libfastpfp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py -x -q > gpurun_out/oc_tests.log 2>&1; echo "tests tot32 rc=$?"; tail -1 gpurun_out/oc_tests.log
for rep in 1 2 3; do for v in "" varlib/var_tot32/libfastpfp.so; do
export FASTPFP_LIB=$v
python - <<'PY'
import sys, os, json, time
sys.path.insert(0, '.')
import bench
for wl in ("c2", "c3"):
    r = bench.secondary_pair(wl)
    print(os.environ.get("FASTPFP_LIB") or "main", wl, r["value"], r.get("ms_per_sweep"), flush=True)
PY
done; done
