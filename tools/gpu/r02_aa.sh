# on-chip projection: back-off between re-polls of stale exchange records
for v in "" varlib/var_ns32/libfastpfp.so varlib/var_ns100/libfastpfp.so varlib/var_ns300/libfastpfp.so ""; do
FASTPFP_LIB=$v timeout 300 python - <<'PY'
import sys, os, json; sys.path.insert(0, ".")
import bench
out = []
for c in ("c2", "c3"):
    r = bench.secondary_pair(c)
    out.append((c, r["value"], r["ms_per_sweep"]))
print(os.environ.get("FASTPFP_LIB") or "main", out)
PY
done
