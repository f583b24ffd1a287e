timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_pg.py tests/test_gpu_ga.py -x -q > gpurun_out/g26_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g26_tests.log
for v in "" varlib/var_oc64/libfastpfp.so; do
FASTPFP_LIB=$v python - <<'PY'
import sys, os, time; sys.path.insert(0, ".")
import bench, json
print(os.environ.get("FASTPFP_LIB"), json.dumps({k: v for k, v in bench.secondary_pair("c1").items() if k in ("value", "solve_ms", "ms_per_sweep", "proj_kernel", "planted_recovery")}))
import torch, paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.planted_unequal(5, 128, 120, d=4, eps1=0.0, eps2=0.0, max_iter1=10, max_iter2=100)
s = F.Solver(p.n, p.n_prime, p.d); s.set_graphs(p.A, p.Ap, p.B, p.Bp)
s.iterate(p.alpha, p.lam, 0, 0, 2, 100, want_x=False); torch.cuda.synchronize()
t0 = time.perf_counter(); s.iterate(p.alpha, p.lam, 0, 0, 10, 100, want_x=False); torch.cuda.synchronize()
print("m=128 10 outer x 100 sweeps:", round((time.perf_counter() - t0) * 1e3, 3), "ms", s.stats()["onchip_tiles"])
PY
done
