# on-chip projection: exact fp64 delta on the integer pipe (no fp64->fp32 conversion per element)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py -x -q > gpurun_out/g32_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g32_tests.log
for v in "" varlib/var_headC/libfastpfp.so "" varlib/var_headC/libfastpfp.so; do
FASTPFP_LIB=$v timeout 300 python - <<'PY'
import sys, os, json; sys.path.insert(0, ".")
import bench
out = []
for c in ("c2", "c3", "c1"):
    r = bench.secondary_pair(c)
    out.append((c, r["value"], r["ms_per_sweep"]))
print(os.environ.get("FASTPFP_LIB") or "main", out)
PY
done
