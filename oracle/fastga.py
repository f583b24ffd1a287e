"""FastGA oracle — plain, slow, float64 CPU transcription of the paper's FastGA (arXiv 1207.1114,
Appendix "FastGA") with slack-padded Sinkhorn normalisation.

TEST INFRASTRUCTURE ONLY (same rules as oracle/fastpfp.py): only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu_baseline / reference legs may import it; the product path never does, and the
two share no code (the seeded generators of `paper_1207_1114_b200/inputs.py` excepted).

What the paper fixes: Graduated Assignment with the Kronecker compatibility
C_aibj = A_ij A'_ab reduces its O(n^4) step `{GAO4}` to the O(n^3) update `{GAO3}`
X^(t+1) = exp(beta A X^(t) A'), followed (as in GA) by Sinkhorn's
alternating row/column normalisation. Everything else is a reading (G1-G8):

  G1  exponent:   Q = A X A' + lambda K  (lambda K inside the exponent so FastGA optimises the same
                  objective as FastPFP; SPEC's design decision). lambda = 0 is the paper's form.
  G2  slack:      m = max(n, n'); the m x m matrix has Q in its top-left n x n' block and slack
                  entries with zero compatibility (Q = 0 there, exp(beta*0) = 1 before stabilisation),
                  re-created at every update (GA slack variables); slack rows when n < n', slack
                  columns when n > n' (as FastPFP's reading A1).
  G3  stabilised exponentiation: each row i of the padded matrix is shifted by its maximum
                  c_i = max_j Q^_ij before exp, E_ij = exp(beta (Q^_ij - c_i)). The first Sinkhorn step
                  is a row normalisation, which divides row i by its sum, so the shift cancels
                  exactly (pinned against the unshifted formula in tests).
  G4  Sinkhorn sweep: one sweep = normalise every row to sum 1, then every column to sum 1 (the
                  paper's "normalizes each row and column ... alternatively").
                  delta_s = max|S^(s) - S^(s-1)| between consecutive sweep outputs; the loop stops at
                  the first s >= 2 with delta_s < eps2, or at s = I_1 (delta_1 is reported as inf:
                  the first sweep has no normalised predecessor).
  G5  annealing:  beta_t = beta0 * rate^t, t = 0, 1, ...; one X update per beta value; the loop
                  runs while beta_t <= beta_max, stops early when rho_t = max|X^(t+1) - X^(t)| < eps1,
                  and never exceeds I_0 updates. Defaults beta0 = 0.5, rate = 1.075, beta_max = 10
                  (conventional GA settings; the paper publishes none).
  G6  X^(t+1) is the top-left n x n' block of the normalised matrix: no blend, no rescale.
  G7  X0 = 1 1^T/(n n') as FastPFP unless given.
  G8  a zero row/column sum cannot occur in exact fp64 for finite Q (every stabilised row holds a 1);
      a column of underflowed entries would divide by 0: the oracle asserts against it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .fastpfp import affinity, gradient

F64 = np.float64

BETA0 = 0.5
BETA_RATE = 1.075
BETA_MAX = 10.0


def gao4_update(A, Ap, X, beta) -> np.ndarray:
    """The O(n^4) GA step `{GAO4}` written with an explicit compatibility tensor
    C[i, a, j, b] = A_ij A'_ab and a quadruple loop: Q_ia = sum_{j,b} C_iajb X_jb,
    X_ia = exp(beta Q_ia). Tiny inputs only: it pins the O(n^3) form `{GAO3}`."""
    A, Ap, X = (np.asarray(M, F64) for M in (A, Ap, X))
    n, n_prime = X.shape
    C = np.zeros((n, n_prime, n, n_prime), dtype=F64)
    for i in range(n):
        for a in range(n_prime):
            for j in range(n):
                for b in range(n_prime):
                    C[i, a, j, b] = A[i, j] * Ap[a, b]
    Q = np.zeros((n, n_prime), dtype=F64)
    for i in range(n):
        for a in range(n_prime):
            s = 0.0
            for j in range(n):
                for b in range(n_prime):
                    s += C[i, a, j, b] * X[j, b]
            Q[i, a] = s
    return np.exp(beta * Q)


def gao3_update(A, Ap, X, beta) -> np.ndarray:
    """`{GAO3}`: X^(t+1) = exp(beta A X^(t) A') (unnormalised, unstabilised)."""
    A, Ap, X = (np.asarray(M, F64) for M in (A, Ap, X))
    return np.exp(beta * (A @ X @ Ap))


def padded_compatibility(Q: np.ndarray, m: int) -> np.ndarray:
    """Q^ (m x m): Q in the top-left block, zero-compatibility slack elsewhere (reading G2)."""
    n, n_prime = Q.shape
    Qh = np.zeros((m, m), dtype=F64)
    Qh[:n, :n_prime] = Q
    return Qh


def stabilised_exp(Qh: np.ndarray, beta: float) -> np.ndarray:
    """E_ij = exp(beta (Q^_ij - max_k Q^_ik)) (reading G3)."""
    Qh = np.asarray(Qh, F64)
    c = np.max(Qh, axis=1, keepdims=True)
    return np.exp(beta * (Qh - c))


def sinkhorn_sweep(S: np.ndarray) -> np.ndarray:
    """One Sinkhorn sweep (reading G4): rows to sum 1, then columns to sum 1."""
    S = np.asarray(S, F64)
    r = S.sum(axis=1, keepdims=True)
    assert np.all(r > 0), "zero row sum (reading G8)"
    R = S / r
    c = R.sum(axis=0, keepdims=True)
    assert np.all(c > 0), "zero column sum (reading G8)"
    return R / c


def sinkhorn_loop(S: np.ndarray, eps2: float, max_iter2: int):
    """Repeat sweeps until delta_s < eps2 (s >= 2) or I_1 sweeps (reading G4).
    Returns (S, sweeps, last_delta)."""
    S = sinkhorn_sweep(S)
    sweeps, delta = 1, float("inf")
    while sweeps < max_iter2:
        Z = sinkhorn_sweep(S)
        delta = float(np.max(np.abs(Z - S)))
        S = Z
        sweeps += 1
        if delta < eps2:
            break
    return S, sweeps, delta


@dataclass
class GAReport:
    iterations: int = 0
    converged: bool = False
    rho: List[float] = field(default_factory=list)
    sweeps: List[int] = field(default_factory=list)
    delta: List[float] = field(default_factory=list)
    beta: List[float] = field(default_factory=list)
    X_trace: List[np.ndarray] = field(default_factory=list)


class FastGA:
    """FastGA state machine: X and the annealing counter t persist across calls, so k calls of
    iterate(max_iter1=1) equal one call with max_iter1=k (the same contract as FastPFP)."""

    def __init__(self, A, Ap, B=None, Bp=None, X0=None, beta0=BETA0, rate=BETA_RATE,
                 beta_max=BETA_MAX):
        self.A = np.asarray(A, F64)
        self.Ap = np.asarray(Ap, F64)
        self.n, self.n_prime = self.A.shape[0], self.Ap.shape[0]
        assert np.array_equal(self.A, self.A.T) and np.array_equal(self.Ap, self.Ap.T)
        self.m = max(self.n, self.n_prime)
        self.K = affinity(B, Bp, self.n, self.n_prime)
        if X0 is None:
            X0 = np.ones((self.n, self.n_prime), dtype=F64) / (self.n * self.n_prime)   # G7
        self.X = np.array(X0, dtype=F64, copy=True)
        self.beta0, self.rate, self.beta_max = float(beta0), float(rate), float(beta_max)
        self.t = 0

    def beta(self, t: int) -> float:
        """beta_t = beta0 * rate^t (reading G5)."""
        return self.beta0 * self.rate ** t

    def outer_step(self, lam, eps2, max_iter2):
        """One FastGA update at beta_t: exponent, stabilised exp, slack-padded Sinkhorn."""
        b = self.beta(self.t)
        Q = gradient(self.A, self.Ap, self.K, self.X, lam)                # G1: A X A' + lambda K
        E = stabilised_exp(padded_compatibility(Q, self.m), b)            # G2, G3
        S, sweeps, delta = sinkhorn_loop(E, eps2, max_iter2)              # G4
        X_new = S[:self.n, :self.n_prime].copy()                          # G6
        rho = float(np.max(np.abs(X_new - self.X)))
        return X_new, rho, sweeps, delta, b

    def iterate(self, lam, eps1, eps2, max_iter1, max_iter2, trace_x=0):
        """Annealing loop (reading G5): while beta_t <= beta_max and fewer than I_0 updates were made
        by this call; stop when rho < eps1."""
        rep = GAReport()
        while rep.iterations < max_iter1 and self.beta(self.t) <= self.beta_max:
            X_new, rho, sweeps, delta, b = self.outer_step(lam, eps2, max_iter2)
            self.X = X_new
            self.t += 1
            rep.iterations += 1
            rep.rho.append(rho)
            rep.sweeps.append(sweeps)
            rep.delta.append(delta)
            rep.beta.append(b)
            if len(rep.X_trace) < trace_x:
                rep.X_trace.append(self.X.copy())
            if rho < eps1:
                rep.converged = True
                break
        return self.X, rep
