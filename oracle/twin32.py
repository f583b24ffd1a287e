"""fp32-storage emulation twin of the oracle — a DIAGNOSTIC, not the oracle (test infrastructure).

Same Algorithm 1 as oracle/fastpfp.py, but every stored matrix (X, Y, the products)
is rounded to float32 the way a GPU path that stores fp32 must round it; the row/column sums and the
P1 correction are evaluated in float64 (the GPU design). It measures how far
ANY fp32-storage implementation drifts from the fp64 oracle on a config before a kernel exists, i.e.
whether the 1e-4 parity tolerance of BASELINE.json is reachable at all (SURVEY.md §7 hard part 1).
"""
from __future__ import annotations

import numpy as np

F32, F64 = np.float32, np.float64


class Twin32:
    def __init__(self, A, Ap, B=None, Bp=None, X0=None, gemm="f32", sweep_arith="f64"):
        self.A = np.asarray(A, F32)
        self.Ap = np.asarray(Ap, F32)
        self.n, self.n_prime = self.A.shape[0], self.Ap.shape[0]
        self.m = max(self.n, self.n_prime)
        if B is None or B.shape[1] == 0:
            self.K = np.zeros((self.n, self.n_prime), F32)
        else:
            self.K = (np.asarray(B, F64) @ np.asarray(Bp, F64).T).astype(F32)
        self.X = (np.full((self.n, self.n_prime), 1.0 / (self.n * self.n_prime), F32)
                  if X0 is None else np.array(X0, F32))
        self.Y = np.zeros((self.m, self.m), F32)
        self.gemm = gemm
        # "f64": every sweep's P1 correction in float64 (the streaming kernel); "f32": only the first
        # sweep after the product, the later ones in float32 (the on-chip kernel)
        self.sweep_arith = sweep_arith

    def _product(self, lam):
        if self.gemm == "f64":   # exact product rounded once to fp32
            G = np.asarray(self.A, F64) @ np.asarray(self.X, F64) @ np.asarray(self.Ap, F64)
            return (G + lam * np.asarray(self.K, F64)).astype(F32)
        U = (self.X @ self.Ap).astype(F32)          # fp32 BLAS accumulation
        return (self.A @ U + F32(lam) * self.K).astype(F32)

    def step(self, lam, alpha, eps2, max_iter2):
        n, npr, m = self.n, self.n_prime, self.m
        self.Y[:n, :npr] = self._product(lam)
        sweeps = 0
        while True:
            Y64 = self.Y.astype(F64)
            r = Y64.sum(1); c = Y64.sum(0); s = r.sum()
            t, u = (1.0 + s / m - r) / m, c / m
            if self.sweep_arith == "f32" and sweeps > 0:
                Z = np.maximum((self.Y + t.astype(F32)[:, None]) - u.astype(F32)[None, :], F32(0))
            else:
                Z = np.maximum(Y64 + t[:, None] - u[None, :], 0.0).astype(F32)
            delta = float(np.max(np.abs(Z - self.Y)))
            self.Y = Z
            sweeps += 1
            if delta < eps2 or sweeps >= max_iter2:
                break
        Xt = ((1.0 - alpha) * self.X.astype(F64) + alpha * self.Y[:n, :npr].astype(F64)).astype(F32)
        mu = float(Xt.max())
        Xn = (Xt.astype(F64) / mu).astype(F32)
        rho = float(np.max(np.abs(Xn - self.X)))
        self.X = Xn
        return rho, sweeps, delta, mu
