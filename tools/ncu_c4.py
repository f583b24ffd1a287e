import sys
sys.path.insert(0, '.')
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs
b = int(sys.argv[1]) if len(sys.argv) > 1 else 148
probs = inputs.config4(batch=8192, first=0, count=b)
s = F.BatchedSolver(b, 128, 128, 0)
s.set_graphs(*inputs.stack_pairs(probs))
X, rep = s.iterate(0.5, 0.0, 0.0, 0.0, 20, 20, want_x=False)
X, rep = s.iterate(0.5, 0.0, 0.0, 0.0, 20, 20, want_x=False)
print("ok")
