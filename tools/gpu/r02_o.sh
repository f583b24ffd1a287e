# tagged-record exchange in the on-chip projection: parity + c2/c3 timing vs the barrier version
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py -x -q > gpurun_out/g27_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g27_tests.log
FASTPFP_LIB=varlib/var_oc512/libfastpfp.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g27_tests512.log 2>&1; echo "tests512 rc=$?"; tail -2 gpurun_out/g27_tests512.log
for v in "" varlib/var_oc512/libfastpfp.so varlib/var_oc64/libfastpfp.so varlib/var_ocprof/libfastpfp.so; do
FASTPFP_LIB=$v timeout 300 python - <<'PY'
import sys, os, json; sys.path.insert(0, ".")
import bench
for c in ("c2", "c3"):
    r = bench.secondary_pair(c)
    print(os.environ.get("FASTPFP_LIB") or "main", c, json.dumps({k: r[k] for k in ("value", "solve_ms", "ms_per_sweep", "total_sweeps")}))
PY
done 2>&1 | grep -v "^oc-prof block" ; FASTPFP_LIB=varlib/var_ocprof/libfastpfp.so timeout 300 python -c "
import sys; sys.path.insert(0, '.'); import bench; bench.secondary_pair('c2')" 2>&1 | grep oc-prof | tail -4
