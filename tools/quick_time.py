"""Quick device timing of the single-pair path (diagnostic)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs

def timeit(p, prec, outer, inner, label):
    s = F.Solver(p.n, p.n_prime, p.d)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.set_x0(p.X0)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, inner, want_x=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, outer, inner, want_x=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label}: prec={prec} {outer} outer x {inner} sweeps: {dt*1e3:.1f} ms total, {dt/outer*1e3:.3f} ms/outer, sweeps={rep.total_sweeps}", flush=True)
    s.close()

which = sys.argv[1:] or ["c2", "c5"]
if "c2" in which:
    p = inputs.config2()
    timeit(p, 2, 5, 300, "c2")
    timeit(p, 2, 5, 1, "c2-gemm-only-ish")
if "c5" in which:
    t0 = time.time(); p = inputs.config5(); print("gen c5", time.time() - t0, flush=True)
    timeit(p, 2, 3, 20, "c5")
    timeit(p, 2, 3, 1, "c5-1sweep")
