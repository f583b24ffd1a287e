# c2/c3 max|X - X_oracle| at termination with 8-byte (default) and 16-byte exchange records for the fp32 sweeps
cat > /tmp/ocerr.py <<'PY'
import sys, os; sys.path.insert(0, '.')
import numpy as np, paper_1207_1114_b200 as F
from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs
for name in ("c2", "c3"):
    p = {"c2": inputs.config2, "c3": inputs.config3}[name]()
    s = F.Solver(p.n, p.n_prime, p.d); s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    if p.X0 is not None: s.set_x0(p.X0)
    X, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2)
    Xo, ro, st = O.solve(p)
    print(os.environ.get("FASTPFP_LIB") or "main(rec8)", name, "max|dX|", float(np.max(np.abs(X.astype(np.float64) - Xo))), "iters", rep.iterations, ro.iterations, flush=True)
PY
for v in "" varlib/var_rec16/libfastpfp.so; do FASTPFP_LIB=$v timeout 900 python /tmp/ocerr.py; done
