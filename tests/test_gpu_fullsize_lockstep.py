"""Lockstep parity at BASELINE.json's full c5 size (configs[4]: n = n' = 16384, d = 64, lambda = 1,
alpha = 0.5, 20 sweeps per outer iteration, eps = 0), in the launch configuration bench.py times.

* `test_c5_full_size_lockstep`: Algorithm 1 from the paper's X0 = 11^T/(nn')
   on the GPU — once with the int8 Ozaki products (the library and bench default) and
  once with 3xTF32 (north_star's named precision) — and in the fp64 oracle, outer iteration by outer
  iteration. After every iteration max|X_gpu - X_oracle| <= 1e-4 (north_star); at the end the
  relative objective difference <= 1e-4 and, when FASTPFP_FULLSIZE_GREEDY=1, >= 99% identical
  greedy assignments. The oracle costs ~1.5 min per outer iteration on the GPU box's 16
  host cores, so the suite runs FASTPFP_FULLSIZE_ITERS (default 3) iterations; the 10-iteration
  record under profiles/ comes from the same test with FASTPFP_FULLSIZE_ITERS=10 and
  FASTPFP_LOCKSTEP_OUT=<json path>.
* `test_c5_full_size_sweep_sums`: the streaming projection computes the row/column sums of a sweep's
  output with fp32 per-lane partials (16 elements of a row, <= 64 rows of a column) and fp64 beyond
  (DESIGN.md §6). Sweep 2 of a 2-sweep launch consumes those sums (and, as every sweep after the
  first of an outer iteration, applies its correction in fp32); it is compared with the oracle's
  fp64 sweep (oracle.sweep = P2(P1(Y))) of the GPU's own sweep-1 output, within the
  bound the fp32 partials and the fp32 correction allow. Nothing here comes from the CUDA path except the values under test.
"""
import json
import os
import time

import numpy as np
import pytest

from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs
from tests.parity import F_RTOL, X_TOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

ITERS = int(os.environ.get("FASTPFP_FULLSIZE_ITERS", "3"))


@pytest.fixture(scope="module")
def c5():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1207_1114_b200 as F
    F.lib()
    return inputs.config5()


def test_c5_full_size_lockstep(c5):
    import paper_1207_1114_b200 as F
    p = c5
    solvers = {}
    for name, prec in (("int8_ozaki", F.PREC_INT8_OZAKI), ("tf32x3", F.PREC_TF32X3)):
        s = F.Solver(p.n, p.n_prime, p.d)
        s.set_option(F.OPT_PRECISION, prec)
        s.set_graphs(p.A, p.Ap, p.B, p.Bp)
        solvers[name] = s
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)
    record = {"workload": "c5 (BASELINE configs[4]) n=n'=16384, d=64, lambda=1, alpha=0.5, 20 sweeps "
                          "per outer, X0 = 11^T/(nn')", "iterations": [], "x_tol": X_TOL}
    for t in range(ITERS):
        t0 = time.perf_counter()
        Xo, ro = st.iterate(p.lam, p.alpha, 0.0, 0.0, 1, p.max_iter2)
        row = {"t": t + 1, "oracle_s": round(time.perf_counter() - t0, 1), "mu_oracle": ro.mu[0],
               "rho_oracle": ro.rho[0]}
        for name, s in solvers.items():
            Xg, rg = s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, p.max_iter2)
            assert rg.sweeps == [p.max_iter2]
            row[name] = {"max_abs_dX": float(np.max(np.abs(Xg.astype(np.float64) - Xo))),
                         "mu": rg.mu[0], "rho": rg.rho[0]}
            del Xg
        record["iterations"].append(row)
        print(json.dumps(row), flush=True)
    f_o = O.objective(st.A, st.Ap, st.K, st.X, p.lam)
    record["objective_oracle"] = f_o
    for name, s in solvers.items():
        f_g = s.objective(p.lam)
        record[f"objective_{name}"] = f_g
        record[f"objective_rel_diff_{name}"] = abs(f_g - f_o) / max(1.0, abs(f_o))
    if os.environ.get("FASTPFP_FULLSIZE_GREEDY") == "1":
        t0 = time.perf_counter()
        a_o = O.greedy_discretize(st.X)
        record["oracle_greedy_s"] = round(time.perf_counter() - t0, 1)
        for name, s in solvers.items():
            a_g = s.discretize()
            record[f"assign_agree_{name}"] = float(np.mean(a_g == a_o))
            record[f"planted_recovery_{name}"] = float(np.mean(a_g == p.perm))
    for s in solvers.values():
        s.close()
    out = os.environ.get("FASTPFP_LOCKSTEP_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(record, f, indent=1)
    print(json.dumps({k: v for k, v in record.items() if k != "iterations"}), flush=True)
    for row in record["iterations"]:
        for name in solvers:
            assert row[name]["max_abs_dX"] <= X_TOL, (row["t"], name, row[name])
    for name in solvers:
        assert record[f"objective_rel_diff_{name}"] <= F_RTOL, (name, record)
        if f"assign_agree_{name}" in record:
            assert record[f"assign_agree_{name}"] >= 0.99, (name, record)


def test_c5_full_size_sweep_sums(c5):
    import paper_1207_1114_b200 as F
    p = c5
    m = p.n
    # Y0: the GPU's projection input after one outer iteration of the bench configuration (a real
    # c5 soft-assignment-shaped matrix, >= 0)
    s = F.Solver(p.n, p.n_prime, p.d)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 1)
    Y0 = torch.from_numpy(s.copy_y()).cuda()
    s.close()
    Y1 = Y0.clone()
    Y2 = Y0.clone()
    F.project(Y1, 0.0, 1)             # sweep 1: sums from the fp64 sums pass
    F.project(Y2, 0.0, 2)             # sweep 2 uses the fp32-per-lane sums of sweep 1's output
    torch.cuda.synchronize()
    y1 = Y1.cpu().numpy().astype(np.float64)
    y2 = Y2.cpu().numpy()
    del Y0, Y1, Y2
    torch.cuda.empty_cache()
    Z, _ = O.sweep(y1)                # the oracle's fp64 sweep of the GPU's stored sweep-1 output
    r, c = y1.sum(1), y1.sum(0)       # y1 >= 0 (P2), so these are also the sums of |y|
    sig = c.sum()
    u = 2.0**-24
    # fp32 partials: row sums over 16-element lane groups (<= 15 u r_i), column sums over <= 64
    # rows (<= 63 u c_j), sigma from the column partials. Sweeps after an outer iteration's first
    # correct in fp32 (checkpointed sweeps): t_i and c_j/m rounded to fp32, then
    # fl(fl(y + t_i) - c_j/m), whose two roundings are <= u (|y| + |t_i| + |c_j/m|) each; the result is
    # stored as computed; x2 margin
    t = (1.0 + sig / m - r) / m
    uc = c / m
    mag = np.abs(y1) + np.abs(t)[:, None] + uc[None, :]
    bound = 2.0 * ((16 * u * r[:, None] + 64 * u * c[None, :] + 64 * u * sig / m) / m
                   + u * (np.abs(t)[:, None] + uc[None, :]) + 2 * u * mag + u * np.abs(Z))
    err = np.abs(y2.astype(np.float64) - Z)
    ratio = float(np.max(err / np.maximum(bound, 1e-300)))
    print(json.dumps({"max_abs_err": float(err.max()), "max_err_over_bound": ratio,
                      "max_bound": float(bound.max())}), flush=True)
    assert ratio <= 1.0, ratio
    # the pin has teeth: dropping one element of a row sum moves that row by y/m >> bound
    i, j = np.unravel_index(int(np.argmax(y1)), y1.shape)
    assert y1[i, j] / m > 10 * bound[i].max()
