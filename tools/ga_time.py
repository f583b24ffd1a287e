"""Time a full FastGA solve at n = 1000 (GA-scaled c2 recipe) through the C-ABI, next to FastPFP c2."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs

p = inputs.ga_pair(2, 1000, d=32, lam=1.0, p=0.5, sigma_e=0.05, eps1=1e-4, eps2=1e-4,
                   max_iter1=300, max_iter2=100)
s = F.Solver(p.n, p.n_prime, p.d)
s.set_option(F.OPT_METHOD, F.METHOD_FASTGA)
s.set_graphs(p.A, p.Ap, p.B, p.Bp)
for rep in range(3):
    s.reset()
    torch.cuda.synchronize()
    t = time.perf_counter()
    X, r = s.iterate(0.0, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2)
    dt = time.perf_counter() - t
    a = s.discretize()
    print(f"FastGA n=1000: {r.iterations} updates, {r.total_sweeps} sweeps, {dt*1e3:.2f} ms "
          f"({dt/r.total_sweeps*1e6:.2f} us/sweep), recovered {np.mean(a == p.perm):.3f}, conv {r.converged}")
