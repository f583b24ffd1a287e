"""Pins for the FastGA oracle (oracle/fastga.py) — values the paper and mathematics
fix, none taken from the CUDA path or from the oracle itself.

* `{GAO3}` equals the O(n^4) GA step `{GAO4}` with C_aibj = A_ij A'_ab,
  written as an explicit compatibility tensor and a quadruple loop.
* Sinkhorn: closed-form 2 x 2 limit, exact one-sweep result on rank-one inputs, fixed
  point on doubly stochastic inputs, and the KL-projection optimality condition of its limit
  (log(D/M) = a 1^T + 1 b^T) checked independently of the iteration.
* Reading G3 (row-max stabilisation) against the unstabilised formula where nothing overflows.
* Reading G5 schedule length; n = 1 trivial run; k calls of iterate(1) = iterate(k);
  planted recovery on small isomorphic pairs.
"""
import math

import numpy as np
import pytest

from oracle import fastga as G
from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs

RNG = np.random.default_rng


def test_gao3_equals_quadruple_loop_gao4():
    # {GAO4} with C_aibj = A_ij A'_ab is {GAO3} (Appendix), random n <= 5
    for seed in range(4):
        r = RNG(seed)
        n, npr = 4, 3 + (seed % 2)
        A = r.random((n, n)); A = A + A.T
        Ap = r.random((npr, npr)); Ap = Ap + Ap.T
        X = r.random((n, npr))
        beta = 0.3 + 0.1 * seed
        np.testing.assert_allclose(G.gao3_update(A, Ap, X, beta), G.gao4_update(A, Ap, X, beta),
                                   rtol=1e-12, atol=0)


def test_sinkhorn_two_by_two_closed_form():
    # the Sinkhorn limit of positive [[a,b],[c,d]] is [[t,1-t],[1-t,t]] with t^2/(1-t)^2 = ad/(bc)
    # (the only doubly stochastic matrix of the form diag(x) M diag(y))
    for seed in range(5):
        a, b, c, d = RNG(10 + seed).random(4) + 0.05
        S, sweeps, delta = G.sinkhorn_loop(np.array([[a, b], [c, d]]), 1e-15, 100000)
        t = math.sqrt(a * d) / (math.sqrt(a * d) + math.sqrt(b * c))
        np.testing.assert_allclose(S, [[t, 1 - t], [1 - t, t]], atol=1e-12)
        assert delta < 1e-15


def test_sinkhorn_rank_one_is_exact_in_one_sweep():
    # a b^T: rows -> 1 b^T / sum(b), columns -> J/m; the second sweep changes nothing (delta = 0)
    r = RNG(3)
    a, b = r.random(5) + 0.1, r.random(5) + 0.1
    S1 = G.sinkhorn_sweep(np.outer(a, b))
    np.testing.assert_allclose(S1, np.full((5, 5), 0.2), atol=1e-15)
    S, sweeps, delta = G.sinkhorn_loop(np.outer(a, b), 1e-12, 50)
    assert sweeps == 2 and delta < 1e-15


def test_sinkhorn_fixed_point_on_doubly_stochastic():
    # a doubly stochastic input (a convex combination of permutations) is a fixed point
    r = RNG(4)
    P = sum(w * np.eye(6)[r.permutation(6)] for w in (0.5, 0.3, 0.2))
    np.testing.assert_allclose(G.sinkhorn_sweep(P), P, atol=1e-15)


def test_sinkhorn_limit_is_kl_projection():
    # the limit D of Sinkhorn on M > 0 is doubly stochastic and log(D/M) = a 1^T + 1 b^T, the
    # first-order condition of min KL(D || M) over doubly stochastic D ("nearest ...
    # under the relative entropy measure"); checked by the double-centring of L = log(D/M)
    for seed in range(3):
        M = RNG(20 + seed).random((7, 7)) + 0.01
        D, _, _ = G.sinkhorn_loop(M, 1e-15, 100000)
        np.testing.assert_allclose(D.sum(0), 1, atol=1e-12)
        np.testing.assert_allclose(D.sum(1), 1, atol=1e-12)
        L = np.log(D / M)
        centred = L - L.mean(0, keepdims=True) - L.mean(1, keepdims=True) + L.mean()
        assert np.max(np.abs(centred)) < 1e-10


def test_stabilisation_cancels_exactly():
    # reading G3: shifting each row by its max before exp changes nothing after the first row
    # normalisation; compare with the unstabilised exp(beta Q^) where it does not overflow
    for (n, npr) in ((5, 5), (4, 6), (6, 4)):
        r = RNG(n * 10 + npr)
        Q = r.random((n, npr)) * 3.0
        m = max(n, npr)
        Qh = G.padded_compatibility(Q, m)
        S_stab, k1, d1 = G.sinkhorn_loop(G.stabilised_exp(Qh, 2.0), 1e-9, 500)
        S_raw, k2, d2 = G.sinkhorn_loop(np.exp(2.0 * Qh), 1e-9, 500)
        np.testing.assert_allclose(S_stab, S_raw, atol=1e-13)
        assert k1 == k2


def test_padded_matrix_slack_is_zero_compatibility():
    # reading G2: the slack region of Q^ is 0, so unstabilised slack entries are exp(0) = 1
    Q = np.arange(6.0).reshape(2, 3)
    Qh = G.padded_compatibility(Q, 3)
    assert np.array_equal(Qh[:2], Q) and np.array_equal(Qh[2], np.zeros(3))
    assert np.array_equal(np.exp(0.7 * Qh)[2], np.ones(3))


def test_schedule_length_and_beta_values():
    # reading G5: beta_t = 0.5 * 1.075^t <= 10 -> t = 0..41 -> 42 updates when eps1 = 0
    p = inputs.ga_pair(7, 8)
    st = G.FastGA(p.A, p.Ap)
    X, rep = st.iterate(0.0, 0.0, 1e-6, 1000, 5)
    assert rep.iterations == 42
    assert rep.beta[0] == 0.5 and rep.beta[-1] == pytest.approx(0.5 * 1.075 ** 41, rel=1e-15)
    assert 0.5 * 1.075 ** 42 > 10.0
    # a further call does nothing (beta_42 > beta_max)
    _, rep2 = st.iterate(0.0, 0.0, 1e-6, 10, 5)
    assert rep2.iterations == 0


def test_single_node_trivial():
    # n = n' = 1 -> X = [[1]]
    st = G.FastGA(np.zeros((1, 1)), np.zeros((1, 1)))
    X, rep = st.iterate(0.0, 1e-6, 1e-6, 5, 5)
    assert X.shape == (1, 1) and X[0, 0] == 1.0


def test_iterates_are_doubly_stochastic_on_the_padded_matrix():
    # every X is the top-left block of a (numerically) doubly stochastic m x m matrix: the
    # smaller-side sums are 1 and the larger-side sums <= 1 at a tight Sinkhorn tolerance
    for (n, npr) in ((6, 6), (5, 8), (8, 5)):
        p = inputs.ga_pair(30 + n, n, npr)
        st = G.FastGA(p.A, p.Ap)
        X, rep = st.iterate(0.0, 0.0, 1e-13, 6, 20000)
        small_axis = 1 if n <= npr else 0
        np.testing.assert_allclose(X.sum(axis=small_axis), 1.0, atol=1e-9)
        assert np.all(X.sum(axis=1 - small_axis) <= 1.0 + 1e-9) and np.all(X >= 0)


def test_k_steps_equal_one_call():
    p = inputs.ga_pair(11, 10)
    a = G.FastGA(p.A, p.Ap)
    Xa, _ = a.iterate(0.0, 0.0, 1e-8, 7, 40)
    b = G.FastGA(p.A, p.Ap)
    for _ in range(7):
        Xb, _ = b.iterate(0.0, 0.0, 1e-8, 1, 40)
    assert np.array_equal(Xa, Xb)


def test_planted_recovery_small_isomorphic():
    # A' = P^T A P, lambda = 0 -> greedy(FastGA) has zero edge error
    ok = 0
    for seed in range(10):
        p = inputs.ga_pair(100 + seed, 12, sigma_e=0.0)
        st = G.FastGA(p.A, p.Ap)
        X, _ = st.iterate(0.0, 1e-6, 1e-6, 100, 100)
        ok += O.edge_error(st.A, st.Ap, O.greedy_discretize(X)) < 1e-9
    assert ok >= 9, ok


def test_planted_recovery_ga_workload_64():
    # the GPU parity workload (n = 64, noisy planted pair) is recovered exactly
    p = inputs.ga_pair(5, 64)
    st = G.FastGA(p.A, p.Ap)
    X, _ = st.iterate(0.0, 1e-6, 1e-6, 100, 100)
    assert np.array_equal(O.greedy_discretize(X), p.perm)


def test_one_sweep_hand_example_rows_then_columns():
    # reading G4, by hand: M = [[1,2],[3,4]] -> rows [[1/3,2/3],[3/7,4/7]] -> columns (sums 16/21,
    # 26/21) -> [[7/16, 7/13], [9/16, 6/13]]; the column step comes last, so columns sum to 1
    S = G.sinkhorn_sweep(np.array([[1.0, 2.0], [3.0, 4.0]]))
    np.testing.assert_allclose(S, [[7 / 16, 7 / 13], [9 / 16, 6 / 13]], rtol=1e-15)
