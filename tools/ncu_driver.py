"""Small driver for ncu captures: sets up a workload and runs `iters` outer iterations."""
import sys
sys.path.insert(0, '.')
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
p = inputs.config5() if wl == "c5" else inputs.config2()
inner = 20
s = F.Solver(p.n, p.n_prime, p.d)
s.set_option(F.OPT_PRECISION, prec)
s.set_graphs(p.A, p.Ap, p.B, p.Bp)
X, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, iters, inner, want_x=False)
print("ok", rep.iterations, rep.total_sweeps)
