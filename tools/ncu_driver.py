"""Small driver for ncu captures and quick device timings (diagnostic only, not a bench value).

    python tools/ncu_driver.py c5|c2|c3|c1 [iters] [precision]   one pair, `iters` outer iterations
    python tools/ncu_driver.py c4 [iters]                         the 8192-pair batch (20 sweeps)
    python tools/ncu_driver.py discretize [n]                     greedy on a converged-looking X
"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_1207_1114_b200 as F  # noqa: E402
from paper_1207_1114_b200 import inputs  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if wl == "c4":
    probs = inputs.config4()
    A, Ap, _, _ = inputs.stack_pairs(probs)
    s = F.BatchedSolver(len(probs), 128, 128, 0)
    s.set_graphs(A, Ap)
    t0 = time.perf_counter()
    s.iterate(0.5, 0.0, 0.0, 0.0, iters, 20, want_x=False)
    print("ok c4", iters, f"{(time.perf_counter() - t0) * 1e3:.1f} ms")
    sys.exit(0)
if wl == "discretize":
    n = iters if len(sys.argv) > 2 else 16384
    s = F.Solver(n, n, 0)
    A = np.zeros((n, n), np.float32)
    s.set_graphs(A, A)
    X0 = inputs.random_matrix(5, n, n, scale=1.0, shift=0.0)
    s.set_x0(np.abs(X0).astype(np.float32))
    for _ in range(3):
        t0 = time.perf_counter()
        a = s.discretize()
        print("ok discretize", n, f"{(time.perf_counter() - t0) * 1e3:.1f} ms")
    sys.exit(0)
prec = int(sys.argv[3]) if len(sys.argv) > 3 else F.PREC_INT8_OZAKI
p = {"c5": inputs.config5, "c2": inputs.config2, "c3": inputs.config3, "c1": inputs.config1}[wl]()
inner = 20
s = F.Solver(p.n, p.n_prime, p.d)
s.set_option(F.OPT_PRECISION, prec)
s.set_graphs(p.A, p.Ap, p.B, p.Bp)
X, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, iters, inner, want_x=False)
print("ok", wl, rep.iterations, rep.total_sweeps)
