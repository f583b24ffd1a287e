"""Shared helpers of the GPU parity tests: run one Problem through the C-ABI (paper_1207_1114_b200)
and through the fp64 oracle on the same seeded inputs, in lockstep, and compare.

Tolerances are BASELINE.json north_star's: max|X_gpu - X_oracle| <= 1e-4 after each of the first
10 outer iterations and at termination, relative objective difference <= 1e-4, >= 99% identical
discretized assignments (identical on planted-permutation cases)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle import fastpfp as O

X_TOL = 1e-4
F_RTOL = 1e-4
ASSIGN_AGREE = 0.99


@dataclass
class PairResult:
    lockstep_max: list
    final_diff: float
    gpu_iters: int
    oracle_iters: int
    gpu_sweeps: list
    oracle_sweeps: list
    f_gpu: float
    f_oracle: float
    assign_gpu: np.ndarray
    assign_oracle: np.ndarray
    X_gpu: np.ndarray
    X_oracle: np.ndarray


def run_pair(p, precision, lockstep=10, slack_mode=0, rescale=1, check_every=None, cta_group=2,
             proj_kernel=0, method=0):
    from paper_1207_1114_b200 import (OPT_CHECK_EVERY, OPT_GEMM_CTA_GROUP, OPT_PRECISION, OPT_RESCALE,
                                      OPT_SLACK_MODE, Solver)
    s = Solver(p.n, p.n_prime, p.d)
    s.set_option(OPT_PRECISION, precision)
    s.set_option(OPT_GEMM_CTA_GROUP, cta_group)
    from paper_1207_1114_b200 import OPT_METHOD, OPT_PROJ_KERNEL
    s.set_option(OPT_PROJ_KERNEL, proj_kernel)
    s.set_option(OPT_METHOD, method)
    s.set_option(OPT_SLACK_MODE, slack_mode)
    s.set_option(OPT_RESCALE, rescale)
    if check_every:
        s.set_option(OPT_CHECK_EVERY, check_every)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.set_x0(p.X0)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0, slack_mode="reset" if slack_mode else "persist",
                   rescale=bool(rescale), method="pg" if method == 1 else "fastpfp")
    lock = []
    g_iters = o_iters = 0
    g_sw, o_sw = [], []
    g_done = o_done = False
    for _ in range(min(lockstep, p.max_iter1)):
        if not g_done:
            Xg, rg = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, 1, p.max_iter2)
            g_iters += rg.iterations; g_sw += rg.sweeps; g_done = rg.converged or rg.degenerate
        if not o_done:
            Xo, ro = st.iterate(p.lam, p.alpha, p.eps1, p.eps2, 1, p.max_iter2)
            o_iters += ro.iterations; o_sw += ro.sweeps; o_done = ro.converged or ro.degenerate
        lock.append(float(np.max(np.abs(Xg.astype(np.float64) - Xo))))
        if g_done and o_done:
            break
    if not g_done and g_iters < p.max_iter1:
        Xg, rg = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1 - g_iters, p.max_iter2)
        g_iters += rg.iterations; g_sw += rg.sweeps
    if not o_done and o_iters < p.max_iter1:
        Xo, ro = st.iterate(p.lam, p.alpha, p.eps1, p.eps2, p.max_iter1 - o_iters, p.max_iter2)
        o_iters += ro.iterations; o_sw += ro.sweeps
    f_g = s.objective(p.lam)
    f_o = O.objective(st.A, st.Ap, st.K, st.X, p.lam)
    a_g = s.discretize()
    a_o = O.greedy_discretize(st.X)
    s.close()
    return PairResult(lock, float(np.max(np.abs(Xg.astype(np.float64) - st.X))), g_iters, o_iters,
                      g_sw, o_sw, f_g, f_o, a_g, a_o, Xg, st.X)


def assert_parity(res: PairResult, planted=None, x_tol=X_TOL):
    assert max(res.lockstep_max) <= x_tol, res.lockstep_max
    assert res.final_diff <= x_tol, res.final_diff
    assert abs(res.f_gpu - res.f_oracle) <= F_RTOL * max(1.0, abs(res.f_oracle)), (res.f_gpu, res.f_oracle)
    agree = float(np.mean(res.assign_gpu == res.assign_oracle))
    assert agree >= ASSIGN_AGREE, agree
    if planted is not None:
        assert np.array_equal(res.assign_gpu, res.assign_oracle)
    assert abs(res.gpu_iters - res.oracle_iters) <= 1, (res.gpu_iters, res.oracle_iters)
