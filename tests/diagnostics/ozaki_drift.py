"""DIAGNOSTIC (test infrastructure): would an Ozaki-scheme int8 GEMM (per-row power-of-two scales,
S signed 7-bit digit slices, exact integer products, digit pairs p + q <= S + 1) keep the fp32 twin
within the 1e-4 parity bound of the fp64 oracle? Emulated exactly in numpy: digit products are
integers < 2^53, so fp64 BLAS computes them exactly; each weight class is rounded to fp32 the way an
int32 TMEM accumulator converted to fp32 would be.

    python -m tests.diagnostics.ozaki_drift c2 12 3
"""
import sys
import time

import numpy as np

from oracle import fastpfp as O
from oracle.twin32 import Twin32
from paper_1207_1114_b200 import inputs

F32, F64 = np.float32, np.float64


def split_rows(M, S):
    """M (rows x K) -> (scale per row, [S] digit matrices), M ~= scale * sum_k D_k 2^-7k."""
    M = np.asarray(M, F64)
    mx = np.max(np.abs(M), axis=1)
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) + 1, 0)
    s = np.exp2(e)
    r = M / s[:, None]
    D = []
    for _ in range(S):
        d = np.clip(np.rint(r * 128.0), -127, 127)
        D.append(d)
        r = r * 128.0 - d
    return s, D


def ozaki_nt(P, Q, S):
    """C = P Q^T via S-slice int8 digits."""
    sP, DP = split_rows(P, S)
    sQ, DQ = split_rows(Q, S)
    C = np.zeros((P.shape[0], Q.shape[0]), F32)
    for w in range(S + 1, 1, -1):            # small weight classes first
        acc = np.zeros_like(C, dtype=F64)
        for p in range(1, S + 1):
            q = w - p
            if 1 <= q <= S:
                acc += DP[p - 1] @ DQ[q - 1].T    # exact integers
        assert np.max(np.abs(acc)) < 2 ** 31
        C = (C + (acc.astype(F32) * F32(2.0 ** (-7 * w)))).astype(F32)
    return (C * sP.astype(F32)[:, None] * sQ.astype(F32)[None, :]).astype(F32)


class TwinOzaki(Twin32):
    def __init__(self, *a, slices=3, **k):
        super().__init__(*a, **k)
        self.S = slices

    def _product(self, lam):
        U = ozaki_nt(self.Ap, self.X, self.S)            # U = A' X^T  (n' x n)
        G = ozaki_nt(self.A, U, self.S)                  # G = A U^T
        return (G + F32(lam) * self.K).astype(F32)


if __name__ == "__main__":
    cfg = sys.argv[1]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    n = int(sys.argv[4]) if len(sys.argv) > 4 else None
    p = inputs.CONFIGS[cfg](n=n) if n else inputs.CONFIGS[cfg]()
    if isinstance(p, list):
        p = p[0]
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)
    tw = TwinOzaki(p.A, p.Ap, p.B, p.Bp, p.X0, slices=S)
    t2 = Twin32(p.A, p.Ap, p.B, p.Bp, p.X0)
    t0 = time.time()
    for t in range(iters):
        X, rep = st.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
        tw.step(p.lam, p.alpha, p.eps2, p.max_iter2)
        t2.step(p.lam, p.alpha, p.eps2, p.max_iter2)
        print(f"t={t:3d} ozaki{S} max|dX|={np.max(np.abs(X - tw.X)):.3e}   fp32 max|dX|="
              f"{np.max(np.abs(X - t2.X)):.3e}   ({time.time() - t0:.1f}s)", flush=True)
    a1, a2 = O.greedy_discretize(X), O.greedy_discretize(tw.X)
    print("assign agree", np.mean(a1 == a2))
