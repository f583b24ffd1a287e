"""SURVEY §8(f4) / paper §6.2: alpha and lambda sensitivity of FastPFP on the synthetic
distance-graph workload, on the GPU (outer iterations, sweeps, solve time, planted-match accuracy,
edge error of the assignment). Writes one JSON document to stdout."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1207_1114_b200 as F
from paper_1207_1114_b200 import inputs


def run(p, alpha, lam):
    s = F.Solver(p.n, p.n_prime, p.d)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, rep = s.iterate(alpha, lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2, want_x=False)
    a = s.discretize()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    acc = float(np.mean(a == p.perm))
    Pm = np.zeros((p.n, p.n_prime)); Pm[np.arange(p.n), a] = 1
    err = float(np.sum((p.A - Pm @ p.Ap @ Pm.T) ** 2))
    s.close()
    return {"alpha": alpha, "lambda": lam, "outer": rep.iterations, "converged": rep.converged,
            "sweeps": rep.total_sweeps, "ms": round(dt * 1e3, 3), "accuracy": acc, "edge_error": err}


out = {"workload": "distance_pair(seed=5, n=1022, dim=3, outliers=0, jitter=0.005, d=128) "
                   "(Stanford-Bunny-sized synthetic 3-D points, P:587, P:611)", "alpha_sweep": [], "lambda_sweep": []}
p = inputs.distance_pair(5, 1022, n_outliers=0, dim=3, jitter=0.005)
for a in [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0]:
    out["alpha_sweep"].append(run(p, a, 10.0))
for lam in [0.0, 1.0, 5.0, 10.0, 50.0]:
    out["lambda_sweep"].append(run(p, 0.5, lam))
print(json.dumps(out, indent=1))
