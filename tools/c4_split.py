"""c4 timing split: 20 outer x {1, 20} sweeps on the 8192-pair batch (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
probs = inputs.config4()
A, Ap, _, _ = inputs.stack_pairs(probs)
s = F.BatchedSolver(8192, 128, 128, 0)
s.set_graphs(A, Ap)
for sw in (1, 5, 20):
    s.set_x0(None); s.iterate(0.5, 0.0, 0.0, 0.0, 2, sw, want_x=False)
    s.set_x0(None); torch.cuda.synchronize(); t = time.perf_counter()
    s.iterate(0.5, 0.0, 0.0, 0.0, 20, sw, want_x=False); torch.cuda.synchronize()
    print(f"c4 20 outer x {sw} sweeps: {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
