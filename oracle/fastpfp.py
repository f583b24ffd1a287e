"""FastPFP oracle — plain, slow, float64 CPU transcription of arXiv 1207.1114.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import anything under `oracle/`. The product path
(`paper_1207_1114_b200/`, the C-ABI library and its CUDA kernels) never imports, links or calls
it, and shares no code with it: the only common module is the seeded input generator
`paper_1207_1114_b200/inputs.py`, which contains none of the method's arithmetic.

Every function cites the PAPER.md line(s) it follows ("P:123" = PAPER.md line 123). The method is
an iteration with a heuristic projection, so the oracle follows Algorithm 1 step by
step, in the paper's order and notation, with the readings listed in DESIGN.md §"Readings"
(SURVEY.md §8(c) A1-A20). Library primitives used as steps: numpy matmul (the products AXA',
BB'^T), sums, max, abs, argsort. No blocking, fusion or reordering beyond the formulas.

Pins (tests/test_oracle_pins.py) fix each function against values that do not come from the oracle
itself: closed forms, worked examples (tests/golden/), brute force and the paper's theorems.
Parity pinning status per function is listed in DESIGN.md §"Oracle pins"; every function below
has at least one pin (none is "parity unpinned").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

F64 = np.float64


# ------------------------------------------------------------------------------------------------
# Problem quantities
# ------------------------------------------------------------------------------------------------

def affinity(B: Optional[np.ndarray], Bp: Optional[np.ndarray], n: int, n_prime: int) -> np.ndarray:
    """K = B B'^T, the n x n' node-affinity matrix ("K denotes the n x n' matrix BB'^T").
    With no attributes (d = 0) K = 0."""
    if B is None or Bp is None or B.shape[1] == 0:
        return np.zeros((n, n_prime), dtype=F64)
    return np.asarray(B, F64) @ np.asarray(Bp, F64).T


def objective(A, Ap, K, X, lam) -> float:
    """f(X) = 1/2 tr(X^T A X A') + lambda tr(X^T K)  (eq. after "note that for")."""
    A, Ap, K, X = (np.asarray(M, F64) for M in (A, Ap, K, X))
    return float(0.5 * np.trace(X.T @ A @ X @ Ap) + lam * np.trace(X.T @ K))


def gradient(A, Ap, K, X, lam) -> np.ndarray:
    """grad f(X) = A X A' + lambda K  (Algorithm 1 line 3)."""
    A, Ap, K, X = (np.asarray(M, F64) for M in (A, Ap, K, X))
    return A @ X @ Ap + lam * K


# ------------------------------------------------------------------------------------------------
# Projections
# ------------------------------------------------------------------------------------------------

def p1_affine(Y: np.ndarray) -> np.ndarray:
    """P1(Y) = Y + (1/n I + 1^T Y 1 / n^2 I - 1/n Y) 1 1^T - 1/n 1 1^T Y   (Algorithm 1 line 5,
    P:389-390; `{P1}` P:300-302 with its 1^T X 1 read as 1^T Y 1, reading A2).

    "n" is the order of the square matrix Y (m = max(n, n'), reading A2). The products with the
    all-ones vector are formed as the paper writes them: Y 1 1^T = (Y 1) 1^T and 1 1^T Y = 1 (1^T Y)."""
    Y = np.asarray(Y, F64)
    m = Y.shape[0]
    assert Y.shape == (m, m), "P1 acts on the square slacked matrix (P:256-266)"
    one = np.ones(m, dtype=F64)
    Y1 = Y @ one                                      # Y 1   (column vector of row sums)
    oneY = one @ Y                                    # 1^T Y (row vector of column sums)
    s = oneY @ one                                    # 1^T Y 1
    term_I = (1.0 / m + s / m**2)                     # (1/n I + 1^T Y 1/n^2 I) 1 1^T: every entry
    term_Y11 = (Y1 / m)[:, None]                      # 1/n Y 1 1^T: entry (i, j) = (Y 1)_i / n
    term_11Y = (oneY / m)[None, :]                    # 1/n 1 1^T Y: entry (i, j) = (1^T Y)_j / n
    return Y + (term_I - term_Y11) - term_11Y


def p2_nonneg(Y: np.ndarray) -> np.ndarray:
    """P2(Y) = (Y + |Y|) / 2   (`{P2}` P:304-305; Algorithm 1 line 6)."""
    Y = np.asarray(Y, F64)
    return (Y + np.abs(Y)) / 2.0


def sweep(Y: np.ndarray):
    """One pass of the successive projection: Z = P2(P1(Y)), and delta = max|Z - Y|
    (inner stopping quantity max(|Y^(t+1) - Y^(t)|), reading A5)."""
    Z = p2_nonneg(p1_affine(Y))
    delta = float(np.max(np.abs(Z - Y))) if Z.size else 0.0
    return Z, delta


def project_loop(Y: np.ndarray, eps2: float, max_iter2: int):
    """Algorithm 1 lines 4-7: repeat {P1; P2} until max|Y^(t+1) - Y^(t)| < eps2 or
    I_1 sweeps were made. At least one sweep; strict '<' (reading A5).
    Returns (Y, sweeps, last_delta)."""
    Y = np.asarray(Y, F64)
    sweeps, delta = 0, float("inf")
    while True:
        Y, delta = sweep(Y)
        sweeps += 1
        if delta < eps2 or sweeps >= max_iter2:
            break
    return Y, sweeps, delta


def slack_embed(X: np.ndarray, m: int, slack: Optional[np.ndarray] = None) -> np.ndarray:
    """Slacked matrix Y with Y_{1:n,1:n'} = X. The extra columns (n > n') or rows
    (n < n', reading A1) hold slack: `slack` (an m x m matrix whose non-X part is used) or 0."""
    n, n_prime = X.shape
    Y = np.zeros((m, m), dtype=F64) if slack is None else np.array(slack, dtype=F64, copy=True)
    Y[:n, :n_prime] = X
    return Y


def pd_project(X: np.ndarray, eps2: float, max_iter2: int):
    """Partial doubly stochastic projection P_d(X) = P_D(Y)_{1:n,1:n'} with fresh zero
    slack, P_D realised by the alternating loop (reading A10).
    Returns (P_d(X), sweeps, delta)."""
    n, n_prime = X.shape
    m = max(n, n_prime)
    Z, sweeps, delta = project_loop(slack_embed(np.asarray(X, F64), m), eps2, max_iter2)
    return Z[:n, :n_prime], sweeps, delta


def dykstra_project(Y: np.ndarray, tol: float = 1e-12, max_iter: int = 100000):
    """DIAGNOSTIC (reading A10): the exact Frobenius projection P_D(Y) of `{DSP}`
     by Dykstra's alternating projection with correction terms between the affine set
    {P1} and the cone {P2}. The paper's loop omits the corrections; with them the
    iteration converges to the nearest doubly stochastic matrix. Not used by the method."""
    Y = np.asarray(Y, F64)
    X = Y.copy()
    Pc = np.zeros_like(Y)      # correction for the affine step (affine sets need none, kept for form)
    Qc = np.zeros_like(Y)      # correction for the cone step
    for _ in range(max_iter):
        Z = p1_affine(X + Pc)
        Pc = X + Pc - Z
        Xn = p2_nonneg(Z + Qc)
        Qc = Z + Qc - Xn
        if np.max(np.abs(Xn - X)) < tol:
            return Xn
        X = Xn
    return X


# ------------------------------------------------------------------------------------------------
# Algorithm 1 with the stopping rules of P:424-427
# ------------------------------------------------------------------------------------------------

@dataclass
class Report:
    """Per-iteration record: rho_t = max|X^(t+1) - X^(t)|, inner sweeps, last inner
    delta, mu_t = max(X~), f(X^(t+1)) (optional)."""
    iterations: int = 0
    converged: bool = False
    degenerate: bool = False
    rho: List[float] = field(default_factory=list)
    sweeps: List[int] = field(default_factory=list)
    delta: List[float] = field(default_factory=list)
    mu: List[float] = field(default_factory=list)
    objective: List[float] = field(default_factory=list)
    X_trace: List[np.ndarray] = field(default_factory=list)


class FastPFP:
    """Algorithm 1 state machine: holds X and Y (slack persists across outer iterations unless
    slack_mode == 'reset', reading A3), so k calls of iterate(max_iter1=1) equal one call with
    max_iter1=k (the C-ABI contract).

    method = "fastpfp" (Algorithm 1, `{fastPFP}` P:206-211) or "pg", the Projected Gradient of
    `{pg}`: X^(t+1) = P_d(X^(t) + alpha grad f(X^(t))) with the same slacked projection,
    initialisation and stopping rules and no blend / rescale (reading A21)."""

    def __init__(self, A, Ap, B=None, Bp=None, X0=None, slack_mode="persist", rescale=True,
                 method="fastpfp"):
        self.A = np.asarray(A, F64)
        self.Ap = np.asarray(Ap, F64)
        self.n, self.n_prime = self.A.shape[0], self.Ap.shape[0]
        assert np.array_equal(self.A, self.A.T) and np.array_equal(self.Ap, self.Ap.T), \
            "undirected graphs: A and A' must be symmetric (P:135-136)"
        self.m = max(self.n, self.n_prime)
        self.K = affinity(B, Bp, self.n, self.n_prime)
        self.slack_mode = slack_mode
        self.rescale = rescale
        assert method in ("fastpfp", "pg")
        self.method = method
        if X0 is None:
            # "X = 1 1^T_{n x n'} / n n', Y = 0_{n x n}" (Algorithm 1 line 1)
            X0 = np.ones((self.n, self.n_prime), dtype=F64) / (self.n * self.n_prime)
        self.X = np.array(X0, dtype=F64, copy=True)
        self.Y = np.zeros((self.m, self.m), dtype=F64)
        self.t = 0

    def outer_step(self, lam, alpha, eps2, max_iter2):
        """One pass of Algorithm 1 lines 3-9. Returns (X_new, rho, sweeps, delta, mu)."""
        n, n_prime = self.n, self.n_prime
        # line 3: Y_{1:n,1:n'} = A X A' + lambda K
        G = gradient(self.A, self.Ap, self.K, self.X, lam)
        if self.slack_mode == "reset":
            self.Y = np.zeros((self.m, self.m), dtype=F64)
        if self.method == "pg":
            # {pg}: project X + alpha grad f; the projection output is the new X
            self.Y[:n, :n_prime] = self.X + alpha * G
            self.Y, sweeps, delta = project_loop(self.Y, eps2, max_iter2)
            X_new = self.Y[:n, :n_prime].copy()
            rho = float(np.max(np.abs(X_new - self.X)))
            return X_new, rho, sweeps, delta, float(np.max(X_new))
        self.Y[:n, :n_prime] = G
        # lines 4-7: repeat P1, P2 until Y converges
        self.Y, sweeps, delta = project_loop(self.Y, eps2, max_iter2)
        # line 8: X = (1 - alpha) X + alpha Y_{1:n,1:n'}
        X_tilde = (1.0 - alpha) * self.X + alpha * self.Y[:n, :n_prime]
        # line 9: X = X / max(X)
        mu = float(np.max(X_tilde))
        if mu <= 1e-300:
            return None, float("nan"), sweeps, delta, mu          # degenerate guard (reading A7)
        X_new = X_tilde / mu if self.rescale else X_tilde
        rho = float(np.max(np.abs(X_new - self.X)))               # P:424-425, after rescale (A6)
        return X_new, rho, sweeps, delta, mu

    def iterate(self, lam, alpha, eps1, eps2, max_iter1, max_iter2, trace_x=0, with_objective=False):
        """Algorithm 1 outer loop: until max|X^(t+1) - X^(t)| < eps1 or I_0 iterations.
        trace_x = number of leading iterates to keep in the report (for lockstep parity)."""
        rep = Report()
        for _ in range(max_iter1):
            X_new, rho, sweeps, delta, mu = self.outer_step(lam, alpha, eps2, max_iter2)
            rep.sweeps.append(sweeps)
            rep.delta.append(delta)
            rep.mu.append(mu)
            if X_new is None:
                rep.degenerate = True
                break
            self.X = X_new
            self.t += 1
            rep.iterations += 1
            rep.rho.append(rho)
            if with_objective:
                rep.objective.append(objective(self.A, self.Ap, self.K, self.X, lam))
            if len(rep.X_trace) < trace_x:
                rep.X_trace.append(self.X.copy())
            if rho < eps1:
                rep.converged = True
                break
        return self.X, rep


def solve(problem, slack_mode="persist", rescale=True, trace_x=0, with_objective=False,
          max_iter1=None, method="fastpfp"):
    """Run Algorithm 1 (or PG) on an `inputs.Problem`. Returns (X, report, state)."""
    st = FastPFP(problem.A, problem.Ap, problem.B, problem.Bp, problem.X0, slack_mode, rescale,
                 method)
    X, rep = st.iterate(problem.lam, problem.alpha, problem.eps1, problem.eps2,
                        problem.max_iter1 if max_iter1 is None else max_iter1, problem.max_iter2,
                        trace_x=trace_x, with_objective=with_objective)
    return X, rep, st


# ------------------------------------------------------------------------------------------------
# Greedy discretization, Algorithm 1 line 11
# ------------------------------------------------------------------------------------------------

def greedy_discretize(X: np.ndarray) -> np.ndarray:
    """Steps 1-3 of P:372-379: repeatedly take the largest X_ij over the live index set L, set
    P_ij = 1 and strike row i and column j; ties go to the smaller row, then the smaller column
    (reading A12). Exactly min(n, n') pairs are taken. Returns assign[i] = j or -1."""
    X = np.asarray(X, F64)
    n, n_prime = X.shape
    assign = np.full(n, -1, dtype=np.int64)
    row_free = np.ones(n, dtype=bool)
    col_free = np.ones(n_prime, dtype=bool)
    # a sort of L by (value desc, row asc, col asc); scanning it is Step 2 repeated
    rows, cols = np.meshgrid(np.arange(n), np.arange(n_prime), indexing="ij")
    order = np.lexsort((cols.ravel(), rows.ravel(), -X.ravel()))
    need = min(n, n_prime)
    taken = 0
    for flat in order:
        i, j = divmod(int(flat), n_prime)
        if row_free[i] and col_free[j]:
            assign[i] = j
            row_free[i] = False
            col_free[j] = False
            taken += 1
            if taken == need:
                break
    return assign


def greedy_discretize_literal(X: np.ndarray) -> np.ndarray:
    """The same Steps 1-3 written with an explicit live set L and argmax (for tiny inputs only);
    used to pin the sort-based version above."""
    X = np.asarray(X, F64)
    n, n_prime = X.shape
    L = {(i, j) for i in range(n) for j in range(n_prime)}
    assign = np.full(n, -1, dtype=np.int64)
    while L:
        best = max(L, key=lambda ij: (X[ij], -ij[0], -ij[1]))
        i_s, j_s = best
        assign[i_s] = j_s
        L = {(i, j) for (i, j) in L if i != i_s and j != j_s}
    return assign


# ------------------------------------------------------------------------------------------------
# Error metrics — reporting only
# ------------------------------------------------------------------------------------------------

def assignment_matrix(assign: np.ndarray, n_prime: int) -> np.ndarray:
    P = np.zeros((assign.size, n_prime), dtype=F64)
    for i, j in enumerate(assign):
        if j >= 0:
            P[i, j] = 1.0
    return P


def edge_error(A, Ap, assign) -> float:
    """||A - X A' X^T||_F^2 at the discrete X."""
    P = assignment_matrix(assign, Ap.shape[0])
    D = np.asarray(A, F64) - P @ np.asarray(Ap, F64) @ P.T
    return float(np.sum(D * D))
