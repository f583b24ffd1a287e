import sys
sys.path.insert(0, '.')
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.config2()
pk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
s = F.Solver(p.n, p.n_prime, p.d)
s.set_option(F.OPT_PROJ_KERNEL, pk)
s.set_graphs(p.A, p.Ap, p.B, p.Bp)
X, rep = s.iterate(p.alpha, p.lam, 0, 0, 2, 50, want_x=False)
print("ok", rep.total_sweeps)
