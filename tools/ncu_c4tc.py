"""One c4 batch launch (tensor-core small-pair kernel) for ncu."""
import sys
sys.path.insert(0, ".")
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
probs = inputs.config4()
A, Ap, _, _ = inputs.stack_pairs(probs)
s = F.BatchedSolver(8192, 128, 128, 0)
s.set_graphs(A, Ap)
s.iterate(0.5, 0.0, 0.0, 0.0, 2, 20, want_x=False)
print("ok")
