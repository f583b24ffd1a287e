"""c2 (n = 1000) per-launch kernel times on the int8 path (diagnostic, run under ncu)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.config2()
s = F.Solver(p.n, p.n_prime, p.d)
s.set_option(F.OPT_PRECISION, F.PREC_INT8_OZAKI)
s.set_graphs(p.A, p.Ap, p.B, p.Bp)
import os
lam = float(os.environ.get('LAM', p.lam))
s.iterate(p.alpha, lam, 0, 0, 3, 300, want_x=False)
torch.cuda.synchronize()
