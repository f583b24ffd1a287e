# on-chip projection variants: rows in flight per warp (unroll), 384 threads; PROF breakdown
for v in "" varlib/var_u1/libfastpfp.so varlib/var_u3/libfastpfp.so varlib/var_u4/libfastpfp.so varlib/var_t384/libfastpfp.so varlib/var_t384u3/libfastpfp.so ""; do
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
FASTPFP_LIB=varlib/var_ocprof/libfastpfp.so timeout 300 python -c "
import sys; sys.path.insert(0, '.'); import bench; bench.secondary_pair('c2')" 2>&1 | grep oc-prof | tail -2
