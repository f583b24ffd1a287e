"""Per-precision device timing of the single-pair path with per-phase split (diagnostic)."""
import sys, time
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
    s.set_option(F.OPT_PROFILE, 1)
    s.reset_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, outer, inner, want_x=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = s.stats()
    print(f"{label}: prec={prec} {outer}x{inner}: {dt/outer*1e3:.3f} ms/outer | gemm {st['gemm_ms']/outer:.3f} ms "
          f"({st['gemm_flops']/st['gemm_ms']/1e9:.1f} TF/s alg) proj {st['proj_ms']/outer:.3f} ms", flush=True)
    s.close()

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
precs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 3]
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
p = inputs.CONFIGS[which](n=n) if n else inputs.CONFIGS[which]()
for prec in precs:
    timeit(p, prec, 3 if which == "c5" else 5, 20 if which == "c5" else 300, which)
