# on-chip projection with an fp32 tile and fp32 sweeps after the first (fp64) one
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py tests/test_gpu_ga.py -x -q > gpurun_out/g34_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/g34_tests.log
for v in "" varlib/var_headE/libfastpfp.so "" varlib/var_headE/libfastpfp.so; do
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
timeout 300 python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import torch, paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
for n in (1500, 2000, 2200):
    p = inputs.planted_unequal(7, n, n, d=8, eps1=0.0, eps2=0.0, max_iter1=3, max_iter2=300)
    for pk in (0, 1):
        s = F.Solver(p.n, p.n_prime, p.d); s.set_option(F.OPT_PROJ_KERNEL, pk); s.set_graphs(p.A, p.Ap, p.B, p.Bp)
        s.iterate(p.alpha, p.lam, 0, 0, 1, 300, want_x=False); torch.cuda.synchronize()
        t0 = time.perf_counter(); s.iterate(p.alpha, p.lam, 0, 0, 3, 300, want_x=False); torch.cuda.synchronize()
        print("m", n, "proj_kernel", pk, "tiles", s.stats()["onchip_tiles"], "us/sweep", round((time.perf_counter() - t0) * 1e6 / 900, 2))
        s.close()
PY
FASTPFP_LIB=varlib/var_ocprof/libfastpfp.so timeout 300 python -c "
import sys; sys.path.insert(0, '.'); import bench; bench.secondary_pair('c2')" 2>&1 | grep oc-prof | tail -2
