# where the c5 e2e time goes: set_graphs (pinned H2D + checks + digits), iterate, copy_x (D2H)
timeout 600 python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch, paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
p = inputs.config5()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
A, Ap, B, Bp = pin(p.A), pin(p.Ap), pin(p.B), pin(p.Bp)
Xh = torch.empty((p.n, p.n_prime), dtype=torch.float32).pin_memory()
s = F.Solver(p.n, p.n_prime, p.d)
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
for r in range(2):
    a = t(lambda: s.set_graphs(A, Ap, B, Bp))
    b = t(lambda: s.set_x0(None))
    c = t(lambda: s.iterate(p.alpha, p.lam, 0.0, 0.0, 20, 20, want_x=False))
    d = t(lambda: s.copy_x(Xh))
    print(f"set_graphs {a:.1f} ms  set_x0 {b:.1f}  iterate {c:.1f}  copy_x {d:.1f}")
dA = torch.empty_like(A, device="cuda")
e = t(lambda: dA.copy_(A, non_blocking=True))
f = t(lambda: Xh.copy_(dA, non_blocking=True))
print(f"torch pinned H2D 1.07 GB {e:.1f} ms ({A.numel()*4/e/1e6:.1f} GB/s), D2H {f:.1f} ms ({A.numel()*4/f/1e6:.1f} GB/s)")
PY
