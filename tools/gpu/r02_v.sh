# where the c2 solve time goes: GEMM vs projection device time per outer iteration, launches
timeout 300 python - <<'PY'
import sys, time, json; sys.path.insert(0, ".")
import torch, paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.config2()
for ce in (4, 1, 8):
    s = F.Solver(p.n, p.n_prime, p.d); s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.set_option(F.OPT_CHECK_EVERY, ce)
    s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False)
    s.set_option(F.OPT_PROFILE, 1)
    ts = []
    for r in range(5):
        s.set_x0(p.X0); s.reset_stats(); torch.cuda.synchronize()
        t0 = time.perf_counter(); X, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    st = s.stats()
    print("check_every", ce, "wall ms", [round(t, 3) for t in ts], "iters", rep.iterations, {k: st[k] for k in ("launches", "gemm_launches", "proj_launches", "gemm_ms", "proj_ms", "outer_iterations")})
    s.set_option(F.OPT_PROFILE, 0)
    ts = []
    for r in range(5):
        s.set_x0(p.X0); torch.cuda.synchronize()
        t0 = time.perf_counter(); X, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print("   no profile wall ms", [round(t, 3) for t in ts])
    s.close()
PY
