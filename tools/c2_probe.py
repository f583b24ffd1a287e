import sys, time, json
sys.path.insert(0, '.')
import torch
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.config2()
for pk in (0, 1, 2):
    s = F.Solver(p.n, p.n_prime, p.d)
    try:
        s.set_option(F.OPT_PROJ_KERNEL, pk)
    except Exception as e:
        print("pk", pk, "error", e); continue
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.iterate(p.alpha, p.lam, 0, 0, 1, 300, want_x=False)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    X, rep = s.iterate(p.alpha, p.lam, 0, 0, 5, 300, want_x=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = s.stats()
    print("pk", pk, "ms/sweep %.4f" % (dt * 1e3 / rep.total_sweeps), {k: st[k] for k in ("onchip_launches", "onchip_tiles", "proj_launches")})
