"""Small end-to-end invocations of every kernel family, for compute-sanitizer (one tool per call):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs

def run(p, prec=0, method=0, pk=0, it=3, sweeps=10):
    s = F.Solver(p.n, p.n_prime, p.d)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_option(F.OPT_METHOD, method)
    s.set_option(F.OPT_PROJ_KERNEL, pk)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    X, r = s.iterate(0.5, p.lam, 1e-6, 1e-6, it, sweeps)
    s.discretize(); s.objective(p.lam)
    s.close()
    print("ok", p.name, prec, method, pk, r.iterations, flush=True)

p1 = inputs.config1()
pu = inputs.planted_unequal(5, 200, 260, d=4)
pw = inputs.planted_unequal(6, 260, 200, d=4)
for prec in (0, 3):
    for pk in (0, 1):
        run(p1, prec, 0, pk); run(pu, prec, 0, pk); run(pw, prec, 0, pk)
    run(inputs.planted_unequal(8, 700, 650, d=4), prec, 0, 2)   # on-chip, 12 x 12 tiles, tagged exchange
    run(pu, prec, 1)                      # PG
    run(inputs.ga_pair(3, 150, 170), prec, 2)   # FastGA
run(p1, 2)                                # SIMT GEMM
b = F.BatchedSolver(4, 64, 64, 0)         # batched small pairs
probs = inputs.config4(n=64, batch=4, fixed=True)
b.set_graphs(*inputs.stack_pairs(probs)); b.iterate(0.5, 0.0, 0.0, 0.0, 2, 5); b.discretize(); b.close()
p5 = inputs.config5(n=256, d=8)          # sharded path at world 1 (NCCL, phase-split projection)
for prec in (0, 3):
    uid = F.nccl_unique_id()              # one id per communicator
    s = F.Solver(256, 256, 8, dist=(0, 1, uid)); s.set_option(F.OPT_PRECISION, prec)
    s.set_graphs(p5.A, p5.Ap, p5.B, p5.Bp); s.iterate(0.5, 1.0, 0.0, 0.0, 2, 5); s.discretize(); s.close()
    print("ok dist", prec, flush=True)
print("all ok")
