"""Measure fp32-twin drift from the fp64 oracle per config (diagnostic; SURVEY §7 hard part 1)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import fastpfp as O
from oracle.twin32 import Twin32
from paper_1207_1114_b200 import inputs

cfg = sys.argv[1]; iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
gemm = sys.argv[3] if len(sys.argv) > 3 else "f32"
p = inputs.CONFIGS[cfg]()
if isinstance(p, list): p = p[0]
st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)
tw = Twin32(p.A, p.Ap, p.B, p.Bp, p.X0, gemm=gemm)
t0 = time.time()
for t in range(iters):
    X, rep = st.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
    rho, s, d, mu = tw.step(p.lam, p.alpha, p.eps2, p.max_iter2)
    diff = np.max(np.abs(X - tw.X))
    print(f"t={t:3d} oracle sweeps={rep.sweeps[0]:4d} rho={rep.rho[0]:.3e} mu={rep.mu[0]:.4f} | twin sweeps={s:4d} rho={rho:.3e} | max|dX|={diff:.3e}  ({time.time()-t0:.1f}s)", flush=True)
    if rep.rho[0] < p.eps1 and rho < p.eps1: break
a1 = O.greedy_discretize(X); a2 = O.greedy_discretize(tw.X)
print("assign agree", np.mean(a1 == a2), "planted", np.mean(a1 == p.perm) if p.perm is not None else None)
