# on-chip projection exchange variants, interleaved c2 timing (separate processes)
for rep in 1; do
for v in "" varlib/var_swC/libfastpfp.so varlib/var_swfC/libfastpfp.so; do
FASTPFP_LIB=$v timeout 300 python - <<'PY' 2>&1 | grep -v "^oc-prof"
import sys, os, json, subprocess; sys.path.insert(0, ".")
import bench
r = bench.secondary_pair("c2")
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
print(os.environ.get("FASTPFP_LIB") or "main", json.dumps({k: r[k] for k in ("value", "ms_per_sweep")}), clk)
PY
done; done
