"""Pins for the fp64 oracle (oracle/fastpfp.py) — values the paper and mathematics fix.

Each test names the PAPER.md passage (P:line) or derivation it pins. None of the expected values
comes from the CUDA path; stored values live in tests/golden/ with their derivation.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs

RNG = np.random.default_rng


# ---------------------------------------------------------------------------------------------
# K, objective, gradient
# ---------------------------------------------------------------------------------------------

def test_affinity_hand_example():
    # B = [[1,0],[0,1]], B' = [[1,0]] -> K = [[1],[0]]  (K = B B'^T)
    K = O.affinity(np.array([[1.0, 0], [0, 1]]), np.array([[1.0, 0]]), 2, 1)
    assert np.array_equal(K, [[1.0], [0.0]])
    assert np.array_equal(O.affinity(None, None, 3, 2), np.zeros((3, 2)))


def test_objective_special_cases():
    # x = 0 -> 0 ; A = A' = I, X = I, lambda = 0 -> 1/2 tr(I) = 1 for n = 2
    I2 = np.eye(2)
    assert O.objective(I2, I2, np.zeros((2, 2)), np.zeros((2, 2)), 3.0) == 0.0
    assert O.objective(I2, I2, np.zeros((2, 2)), I2, 0.0) == pytest.approx(1.0, abs=1e-15)


def test_objective_quadruple_loop():
    # f(X) = sum_{i,j,a,b} 1/2 X_ia A_ij X_jb A'_ab + lambda sum_{i,a} X_ia K_ia (the elementwise
    # expansion of 1/2 tr(X^T A X A') + lambda tr(X^T K)) on random 4 x 3 instances
    for seed in range(5):
        r = RNG(seed)
        n, npr = 4, 3
        A = r.random((n, n)); A = A + A.T
        Ap = r.random((npr, npr)); Ap = Ap + Ap.T
        K = r.standard_normal((n, npr)); X = r.random((n, npr)); lam = 0.7
        ref = 0.0
        for i, j, a, b in itertools.product(range(n), range(n), range(npr), range(npr)):
            ref += 0.5 * X[i, a] * A[i, j] * X[j, b] * Ap[a, b]
        for i, a in itertools.product(range(n), range(npr)):
            ref += lam * X[i, a] * K[i, a]
        assert O.objective(A, Ap, K, X, lam) == pytest.approx(ref, rel=1e-12, abs=1e-12)


def test_gradient_finite_differences():
    # grad f = A X A' + lambda K vs central differences of f, step 1e-5
    for seed in range(5):
        r = RNG(100 + seed)
        n, npr = 5, 4
        A = r.random((n, n)); A = A + A.T
        Ap = r.random((npr, npr)); Ap = Ap + Ap.T
        K = r.standard_normal((n, npr)); X = r.random((n, npr)); lam = 1.3
        G = O.gradient(A, Ap, K, X, lam)
        h = 1e-5
        for i, a in itertools.product(range(n), range(npr)):
            Xp = X.copy(); Xp[i, a] += h
            Xm = X.copy(); Xm[i, a] -= h
            fd = (O.objective(A, Ap, K, Xp, lam) - O.objective(A, Ap, K, Xm, lam)) / (2 * h)
            assert G[i, a] == pytest.approx(fd, abs=1e-6, rel=1e-6)


def test_gradient_special_cases():
    r = RNG(7)
    A = r.random((4, 4)); A = A + A.T
    K = r.standard_normal((4, 4))
    # x = 0 -> lambda K ; lambda = 0, A' = I, X = I -> A
    assert np.allclose(O.gradient(A, A, K, np.zeros((4, 4)), 2.0), 2.0 * K, atol=0)
    assert np.array_equal(O.gradient(A, np.eye(4), K, np.eye(4), 0.0), A)


# ---------------------------------------------------------------------------------------------
# P1 / P2 (derivation P:743-761)
# ---------------------------------------------------------------------------------------------

def _lstsq_affine_projection(Y):
    """argmin ||D - Y||_F s.t. D 1 = 1, D^T 1 = 1 via the KKT system (independent of {P1})."""
    m = Y.shape[0]
    # constraint matrix C vec(D) = 1 (row sums, then column sums); vec is row-major
    C = np.zeros((2 * m, m * m))
    for i in range(m):
        C[i, i * m:(i + 1) * m] = 1.0
        C[m + i, i::m] = 1.0
    y = Y.ravel()
    # minimise ||d - y||^2 s.t. C d = 1  ->  d = y - C^T w,  C C^T w = C y - 1 (least squares)
    w, *_ = np.linalg.lstsq(C @ C.T, C @ y - 1.0, rcond=None)
    return (y - C.T @ w).reshape(m, m)


def test_p1_is_exact_affine_projection():
    # {P1} (with 1^T Y 1, reading A2) is the orthogonal projection onto
    # {D 1 = 1, D^T 1 = 1} -- including for asymmetric Y
    for seed, m in [(0, 3), (1, 4), (2, 7), (3, 10)]:
        Y = RNG(seed).standard_normal((m, m)) * 5
        Z = O.p1_affine(Y)
        assert np.allclose(Z, _lstsq_affine_projection(Y), atol=1e-12)
        assert np.allclose(Z.sum(1), 1.0, atol=1e-12) and np.allclose(Z.sum(0), 1.0, atol=1e-12)
        assert np.allclose(O.p1_affine(Z), Z, atol=1e-12)           # idempotent


def test_p1_of_zero_and_doubly_stochastic():
    m = 5
    assert np.allclose(O.p1_affine(np.zeros((m, m))), np.full((m, m), 1 / m), atol=1e-15)
    P = np.eye(m)[RNG(0).permutation(m)]
    assert np.allclose(O.p1_affine(P), P, atol=1e-15)


def test_p2_hand_example():
    # [[-1,2],[0,-3]] -> [[0,2],[0,0]]; idempotent   ({P2})
    Z = O.p2_nonneg(np.array([[-1.0, 2.0], [0.0, -3.0]]))
    assert np.array_equal(Z, [[0.0, 2.0], [0.0, 0.0]])
    assert np.array_equal(O.p2_nonneg(Z), Z)


def test_dyadic_sweep_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "dyadic_sweep.json")))
    Y0 = np.array(g["Y0"])
    Z, d = O.sweep(Y0)
    assert np.array_equal(Z, g["sweep1"]["Z"]) and d == g["sweep1"]["delta"]
    for c in g["cases"]:
        Y, s, d = O.project_loop(Y0, c["eps2"], c["max_iter2"])
        assert s == c["sweeps"]
        assert np.array_equal(Y, np.diag([c["diag"]] * 2))
        assert d == c["delta"]


def test_two_by_two_limit_closed_form():
    # For m = 2 the DS polytope is {t I + (1-t) J'}; the projection is
    # t = clamp((Y11 + Y22 - Y12 - Y21 + 2)/4, 0, 1); the alternating loop reaches it
    # because the affine set is a line (P:308-311 holds here).
    r = RNG(11)
    anti = np.array([[0.0, 1.0], [1.0, 0.0]])
    for _ in range(50):
        Y = r.standard_normal((2, 2)) * 3
        t = np.clip((Y[0, 0] + Y[1, 1] - Y[0, 1] - Y[1, 0] + 2) / 4, 0, 1)
        Z, s, d = O.project_loop(Y, 1e-14, 10000)
        assert np.allclose(Z, t * np.eye(2) + (1 - t) * anti, atol=1e-12)
    Z, _, _ = O.project_loop(np.array([[2.0, 0.0], [0.0, 0.0]]), 1e-14, 100)
    assert np.array_equal(Z, np.eye(2))


# ---------------------------------------------------------------------------------------------
# P_d properties (Lemma 1)
# ---------------------------------------------------------------------------------------------

def _smaller_larger_sums(X):
    n, npr = X.shape
    if n >= npr:
        return X.sum(0), X.sum(1)     # X^T 1 = 1 (smaller side n'), X 1 <= 1
    return X.sum(1), X.sum(0)


@pytest.mark.parametrize("n,npr", [(6, 4), (4, 6), (5, 5), (12, 7), (9, 16)])
def test_pd_feasibility_and_idempotence(n, npr):
    # P_d output is partial doubly stochastic within 1e-9 at tight eps2 (BJ north star);
    # one more sweep on the converged slacked matrix moves it by <= 1e-9 (idempotence of P_D,
    # P:308-313). (Re-embedding the n x n' block with *zero* slack is not idempotent: the slack
    # construction of P:256-266 only realises P_d through the persistent slack.)
    for seed in range(5):
        X = RNG(seed * 31 + n).standard_normal((n, npr)) * 2 + 0.3
        m = max(n, npr)
        Y, s, d = O.project_loop(O.slack_embed(X, m), 1e-13, 200000)
        D = Y[:n, :npr]
        small, large = _smaller_larger_sums(D)
        assert np.all(Y >= -1e-9)
        assert np.allclose(small, 1.0, atol=1e-9)
        assert np.all(large <= 1.0 + 1e-9)
        Y2, d2 = O.sweep(Y)
        assert d2 <= 1e-9


def test_pd_nonexpansive_fixed_sweeps():
    # Lemma 1: ||P_d(X1) - P_d(X2)||_F <= ||X1 - X2||_F. With a fixed sweep count the
    # map is a composition of projections onto convex sets, hence nonexpansive exactly.
    r = RNG(5)
    for k in range(200):
        n = int(r.integers(2, 9)); npr = int(r.integers(2, 9))
        X1 = r.standard_normal((n, npr)); X2 = X1 + r.standard_normal((n, npr)) * r.random()
        for sweeps in (1, 3, 10):
            P1, _, _ = O.pd_project(X1, 0.0, sweeps)
            P2, _, _ = O.pd_project(X2, 0.0, sweeps)
            assert np.linalg.norm(P1 - P2) <= np.linalg.norm(X1 - X2) + 1e-9


def test_alternation_fejer_monotone():
    # each P1 or P2 step never increases the distance to a fixed feasible point
    r = RNG(9)
    m = 6
    F = np.eye(m)[r.permutation(m)] * 0.5 + np.full((m, m), 0.5 / m)   # doubly stochastic
    Y = r.standard_normal((m, m)) * 3
    dist = np.linalg.norm(Y - F)
    for _ in range(30):
        Y = O.p1_affine(Y); d1 = np.linalg.norm(Y - F); assert d1 <= dist + 1e-12; dist = d1
        Y = O.p2_nonneg(Y); d2 = np.linalg.norm(Y - F); assert d2 <= dist + 1e-12; dist = d2


# ---------------------------------------------------------------------------------------------
# Algorithm 1
# ---------------------------------------------------------------------------------------------

def test_dyadic_two_node_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "dyadic_two_node.json")))
    st = O.FastPFP(np.array(g["A"]), np.array(g["Ap"]), np.array(g["B"]), np.array(g["Bp"]),
                   np.array(g["X0"]))
    for t, it in enumerate(g["iters"]):
        G = O.gradient(st.A, st.Ap, st.K, st.X, g["lam"])
        assert np.array_equal(G, it["G"])
        Z1, d1 = O.sweep(G)
        assert np.array_equal(Z1, it["sweep1_Z"]) and d1 == it["sweep1_delta"]
        X, rep = st.iterate(g["lam"], g["alpha"], 0.0, g["eps2"], 1, g["max_iter2"])
        assert rep.sweeps == [it["sweeps"]] and rep.mu == [it["mu"]]
        if "X_rtol" in it:
            assert np.allclose(X, it["X"], rtol=it["X_rtol"], atol=0)
        else:
            assert np.array_equal(X, it["X"]) and rep.rho == [it["rho"]]
        if "last_delta" in it:
            assert rep.delta == [it["last_delta"]]
    assert list(O.greedy_discretize(st.X)) == g["assignment"]


def test_single_node_trivial():
    # n = n' = 1: Y = [[0]] -> P1 gives [[1]]; X = [[1]] with rho = 0 at t = 0
    X, rep, _ = O.solve(inputs.Problem("one", np.zeros((1, 1), np.float32), np.zeros((1, 1), np.float32),
                                       None, None, 0.0, 0.5, 1e-6, 1e-6, 10, 10))
    assert np.array_equal(X, [[1.0]]) and rep.converged and rep.iterations == 1 and rep.rho == [0.0]


def test_k_steps_equal_one_call():
    # checkpoint/resume invariant: k x iterate(1) == iterate(k), slack persisting
    p = inputs.random_problem(3, 9, 6, d=2, lam=0.5, max_iter1=7, max_iter2=20)
    a = O.FastPFP(p.A, p.Ap, p.B, p.Bp)
    Xa, _ = a.iterate(p.lam, p.alpha, 0.0, p.eps2, 7, p.max_iter2)
    b = O.FastPFP(p.A, p.Ap, p.B, p.Bp)
    for _ in range(7):
        Xb, _ = b.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
    assert np.array_equal(Xa, Xb)


@pytest.mark.parametrize("slack_mode", ["persist", "reset"])
def test_transpose_equivariance(slack_mode):
    # Reading A1: padding the smaller side with slack rows (n < n') equals solving the swapped
    # problem (A', A, K^T) with slack columns and transposing (P1/P2 are transpose-equivariant).
    p = inputs.random_problem(4, 7, 11, d=3, lam=0.8, eps1=0.0, eps2=1e-6, max_iter1=8, max_iter2=40)
    X1, r1, _ = O.solve(p, slack_mode=slack_mode)
    q = inputs.Problem("swap", p.Ap, p.A, p.Bp, p.B, p.lam, p.alpha, p.eps1, p.eps2,
                       p.max_iter1, p.max_iter2)
    X2, r2, _ = O.solve(q, slack_mode=slack_mode)
    assert np.allclose(X1, X2.T, atol=1e-12) and r1.sweeps == r2.sweeps


def test_relabel_equivariance():
    # permuting A, A', K consistently permutes X
    p = inputs.random_problem(5, 8, 6, d=2, lam=0.3, eps1=0.0, eps2=1e-7, max_iter1=6, max_iter2=30)
    X1, _, _ = O.solve(p)
    r = RNG(1)
    s = r.permutation(8); t = r.permutation(6)
    q = inputs.Problem("perm", p.A[np.ix_(s, s)], p.Ap[np.ix_(t, t)], p.B[s], p.Bp[t], p.lam,
                       p.alpha, p.eps1, p.eps2, p.max_iter1, p.max_iter2)
    X2, _, _ = O.solve(q)
    assert np.allclose(X2, X1[np.ix_(s, t)], atol=1e-12)


@pytest.mark.parametrize("n,npr", [(10, 6), (6, 10), (8, 8)])
def test_smaller_side_sum_recursion(n, npr):
    # Alg. 1 lines 8-9 with the P1 constraint: the smaller-side sums s_t
    # obey s_{t+1} = ((1-alpha) s_t + alpha (1 + e_t)) / mu_t, e_t = feasibility error of the
    # projection output; with a uniform X0 all entries of s_t stay equal up to sum|e|.
    p = inputs.random_problem(6, n, npr, d=2, lam=1.0, eps1=0.0, eps2=1e-12, max_iter1=6,
                              max_iter2=5000)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp)
    ax = 1 if n <= npr else 0
    s = st.X.sum(axis=ax)
    for _ in range(6):
        X, rep = st.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
        Zs = st.Y[:n, :npr].sum(axis=ax)
        s_pred = ((1 - p.alpha) * s + p.alpha * Zs) / rep.mu[0]
        assert np.allclose(X.sum(axis=ax), s_pred, atol=1e-12)
        assert np.max(np.abs(Zs - 1.0)) < 1e-8
        s = X.sum(axis=ax)
        assert np.ptp(s) < 1e-7


def test_convex_combination_closure_without_rescale():
    # with a partial-DS X0 and rescale off, every iterate stays partial DS (A20)
    n, npr = 9, 6
    p = inputs.random_problem(8, n, npr, d=2, lam=0.5, eps1=0.0, eps2=1e-13, max_iter1=8,
                              max_iter2=100000)
    X0 = np.full((n, npr), 1.0 / n)             # column sums 1, row sums n'/n <= 1
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, X0, rescale=False)
    for _ in range(8):
        X, _ = st.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
        assert np.all(X >= -1e-9)
        assert np.allclose(X.sum(0), 1.0, atol=1e-9) and np.all(X.sum(1) <= 1 + 1e-9)


def test_theorem1_rate():
    # Theorem 1: with ||A (x) A'||_2 = eps = 0.5, rescale off (A11), alpha = 0.5,
    # ||dX^(t+1)|| / ||dX^(t)|| <= 1 - alpha + alpha eps = 0.75 (+0.05 slack)
    n = 50
    r = RNG(12)
    A = r.random((n, n)); A = (A + A.T) / 2; np.fill_diagonal(A, 0)
    Ap = r.random((n, n)); Ap = (Ap + Ap.T) / 2; np.fill_diagonal(Ap, 0)
    A = A / np.linalg.norm(A, 2) * np.sqrt(0.5)
    Ap = Ap / np.linalg.norm(Ap, 2) * np.sqrt(0.5)
    assert np.linalg.norm(A, 2) * np.linalg.norm(Ap, 2) == pytest.approx(0.5, rel=1e-12)
    st = O.FastPFP(A, Ap, rescale=False)
    prev, ratios = None, []
    Xprev = st.X.copy()
    for t in range(40):
        X, _ = st.iterate(0.0, 0.5, 0.0, 1e-14, 1, 100000)
        d = np.linalg.norm(X - Xprev); Xprev = X.copy()
        if prev is not None and prev > 1e-12:
            ratios.append(d / prev)
        prev = d
    assert max(ratios[5:]) <= 0.80


def test_fixed_point_form_at_termination():
    # at a fixed point mu X = (1 - alpha) X + alpha Z, so X ~ Z / max Z
    p = inputs.random_problem(13, 12, 12, d=2, lam=1.0, eps1=1e-9, eps2=1e-12, max_iter1=2000,
                              max_iter2=10000)
    X, rep, st = O.solve(p)
    assert rep.converged
    Z = st.Y[:12, :12]
    assert np.max(np.abs(X - Z / Z.max())) < 1e-6


# ---------------------------------------------------------------------------------------------
# Greedy discretization
# ---------------------------------------------------------------------------------------------

def test_greedy_hand_example():
    # [[0.9, 0.8], [0.7, 0.1]] -> picks 0.9 then 0.1 -> identity (greedy != LAP optimum)
    assert list(O.greedy_discretize(np.array([[0.9, 0.8], [0.7, 0.1]]))) == [0, 1]


def test_greedy_matches_literal_steps():
    r = RNG(21)
    for _ in range(30):
        n, npr = int(r.integers(1, 7)), int(r.integers(1, 7))
        X = np.round(r.random((n, npr)) * 4) / 4        # many ties
        assert np.array_equal(O.greedy_discretize(X), O.greedy_discretize_literal(X))


def test_greedy_permutation_equivariance_and_fixed_points():
    r = RNG(22)
    P = np.eye(7)[r.permutation(7)]
    assert np.array_equal(O.greedy_discretize(P), np.argmax(P, 1))
    X = r.random((7, 5))
    a = O.greedy_discretize(X)
    s, t = r.permutation(7), r.permutation(5)
    b = O.greedy_discretize(X[np.ix_(s, t)])
    tinv = np.argsort(t)
    for k in range(7):
        expect = a[s[k]]
        assert b[k] == (-1 if expect < 0 else tinv[expect])
    assert (a >= 0).sum() == 5 and len(set(a[a >= 0])) == 5


# ---------------------------------------------------------------------------------------------
# Whole method vs the global optimum (BJ north star)
# ---------------------------------------------------------------------------------------------

def test_brute_force_small():
    # for n <= 7, f(FastPFP + greedy) <= max over all permutations of f; count optimum hits
    hits = 0
    trials = 20
    for seed in range(trials):
        n = 6
        p = inputs.random_problem(100 + seed, n, n, d=2, lam=0.5, eps1=1e-6, eps2=1e-8,
                                  max_iter1=300, max_iter2=2000)
        X, _, st = O.solve(p)
        a = O.greedy_discretize(X)
        f_alg = O.objective(st.A, st.Ap, st.K, O.assignment_matrix(a, n), p.lam)
        best = max(O.objective(st.A, st.Ap, st.K, np.eye(n)[list(perm)], p.lam)
                   for perm in itertools.permutations(range(n)))
        assert f_alg <= best + 1e-9
        hits += f_alg >= best - 1e-9
    assert hits >= 12, hits   # S:511 expects >= 15/20 on its n=4 instances; recorded in DESIGN.md


def test_planted_recovery_config1():
    # BJ configs[0]: noiseless planted isomorphism, n = 64 -> greedy recovers P
    p = inputs.config1()
    X, rep, st = O.solve(p)
    a = O.greedy_discretize(X)
    assert np.array_equal(a, p.perm) or O.edge_error(st.A, st.Ap, a) == 0.0


@pytest.mark.slow
def test_planted_recovery_unweighted_e1():
    # E1 case (a): unweighted n = 100, 50% connectivity, isomorphic -> excess error 0
    ok = 0
    for seed in range(10):
        r = RNG(500 + seed)
        n = 100
        up = np.triu((r.random((n, n)) < 0.5).astype(np.float32), 1)
        A = up + up.T
        pi = r.permutation(n)
        Ap = inputs.relabel(A, pi)
        p = inputs.Problem("e1", A, Ap, None, None, 0.0, 0.5, 1e-4, 1e-4, 300, 300)
        X, _, st = O.solve(p)
        ok += O.edge_error(st.A, st.Ap, O.greedy_discretize(X)) == 0.0
    assert ok >= 9


# ---------------------------------------------------------------------------------------------
# Projected Gradient {pg}, SURVEY §8(f2)
# ---------------------------------------------------------------------------------------------

def test_pg_dyadic_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "dyadic_pg.json")))
    st = O.FastPFP(np.array(g["A"]), np.array(g["Ap"]), np.array(g["B"]), np.array(g["Bp"]),
                   np.array(g["X0"]), method="pg")
    for it in g["iters"]:
        X, rep = st.iterate(g["lam"], g["alpha"], 0.0, g["eps2"], 1, g["max_iter2"])
        assert np.array_equal(X, it["X"]) and rep.sweeps == [it["sweeps"]] and rep.rho == [it["rho"]]


@pytest.mark.parametrize("n,npr", [(12, 8), (8, 12), (10, 10)])
def test_pg_iterates_are_partial_doubly_stochastic(n, npr):
    # every PG iterate is a P_d output, so it is partial DS at tight eps2
    p = inputs.random_problem(31 + n, n, npr, d=2, lam=0.5, eps1=0.0, eps2=1e-13, max_iter1=6,
                              max_iter2=200000)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, method="pg")
    for _ in range(6):
        X, _ = st.iterate(p.lam, 0.01, 0.0, p.eps2, 1, p.max_iter2)
        small, large = _smaller_larger_sums(X)
        assert np.all(X >= -1e-9) and np.allclose(small, 1.0, atol=1e-9) and np.all(large <= 1 + 1e-9)


def test_pg_zero_gradient_is_projection_fixed_point():
    # A = A' = 0, lambda = 0: grad f = 0, so X1 = P_d(X0) and X2 = P_d(X1) = X1 (idempotence)
    n = 7
    st = O.FastPFP(np.zeros((n, n)), np.zeros((n, n)), method="pg")
    X1, _ = st.iterate(0.0, 0.5, 0.0, 1e-14, 1, 100000)
    X2, rep = st.iterate(0.0, 0.5, 0.0, 1e-14, 1, 100000)
    assert np.allclose(X1, np.full((n, n), 1.0 / n), atol=1e-12) and rep.rho[0] < 1e-12


# ---------------------------------------------------------------------------------------------
# distance-graph workload and the Dykstra diagnostic
# ---------------------------------------------------------------------------------------------

def test_distance_pair_planted_geometry():
    # the partner is a rigid motion of the points: inlier distances are preserved up to the jitter
    p = inputs.distance_pair(3, 40, n_outliers=5, dim=3, jitter=0.0)
    Ainl = p.Ap[np.ix_(p.perm, p.perm)]
    assert np.allclose(Ainl, p.A, atol=1e-5)
    assert np.array_equal(p.A, p.A.T) and np.array_equal(p.Ap, p.Ap.T)
    assert np.allclose(np.linalg.norm(p.B, axis=1), 1.0, atol=1e-5) and np.all(p.B >= 0)


def test_distance_pair_recovered_by_fastpfp():
    # fully connected distance graphs + unit 128-d attributes: with lambda = 10 (the unit attributes
    # carry ~1/10 of SIFT's inner-product scale) the planted match of the inliers is found
    p = inputs.distance_pair(11, 40, n_outliers=6, dim=2, jitter=0.002, lam=10.0)
    X, rep, st = O.solve(p)
    a = O.greedy_discretize(X)
    assert rep.converged and np.mean(a == p.perm) >= 0.95


def test_dykstra_is_exact_projection_and_closer_than_alternation():
    # Dykstra reaches the nearest DS matrix: it satisfies the KKT optimality of {DSP}:
    # Y - D = a 1^T + 1 b^T - N with N >= 0 supported where D = 0 (checked via a 2x2 closed form and
    # by being no farther from Y than the plain alternating limit)
    r = RNG(17)
    for _ in range(20):
        Y = r.standard_normal((2, 2)) * 3
        t = np.clip((Y[0, 0] + Y[1, 1] - Y[0, 1] - Y[1, 0] + 2) / 4, 0, 1)
        anti = np.array([[0.0, 1.0], [1.0, 0.0]])
        assert np.allclose(O.dykstra_project(Y), t * np.eye(2) + (1 - t) * anti, atol=1e-9)
    for _ in range(10):
        Y = r.standard_normal((6, 6)) * 2
        D = O.dykstra_project(Y, tol=1e-13)
        A, _, _ = O.project_loop(Y, 1e-13, 200000)
        assert np.allclose(D.sum(0), 1, atol=1e-8) and np.allclose(D.sum(1), 1, atol=1e-8)
        assert np.all(D >= -1e-10)
        assert np.linalg.norm(Y - D) <= np.linalg.norm(Y - A) + 1e-9


def test_edge_error_hand_examples():
    """||A - X A' X^T||_F^2 at a discrete X, values worked by hand.
    A is the weighted path 0-1-2 (weights 1, 2); A' is the same path with the weights swapped.
    Identity assignment: entries (0,1), (1,0) differ by 1 and (1,2), (2,1) by 1 -> 4.
    Reversal 0->2, 1->1, 2->0 maps A' onto A exactly -> 0. Unequal sizes: A = [[0,3],[3,0]],
    A' = [[0]], row 1 unmatched (-1) -> both off-diagonal 3s are unexplained -> 18."""
    A = np.array([[0, 1, 0], [1, 0, 2], [0, 2, 0]], float)
    Ap = np.array([[0, 2, 0], [2, 0, 1], [0, 1, 0]], float)
    assert O.edge_error(A, Ap, np.array([0, 1, 2])) == 4.0
    assert O.edge_error(A, Ap, np.array([2, 1, 0])) == 0.0
    assert O.edge_error(np.array([[0, 3], [3, 0]], float), np.zeros((1, 1)), np.array([0, -1])) == 18.0
