"""Seeded synthetic inputs for FastPFP (arXiv 1207.1114) — shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no gradient, no projection, no K = BB'^T,
no rescale, no discretization): it only draws the graphs, attributes, planted permutation and
solver hyper-parameters that both sides consume. It is the one module the oracle (`oracle/`)
and the CUDA path (`paper_1207_1114_b200/`) may both import.

Recipe (DESIGN.md §"Input recipe"); the paper's §5.1 protocol (PAPER.md:437-446:
random graphs, planted permutation, edge noise, node deletion) restated on weighted graphs:

* A is symmetric with a zero diagonal; each upper-triangle pair is an edge with probability p and
  weight U(0,1) (BASELINE.json configs; the paper's §5.1 graphs are 0/1 with p = 0.5).
* A planted permutation pi (uniform) relabels a noisy copy: A'[pi(i), pi(j)] = A[i, j] + E[i, j],
  i.e. A' = P^T (A + E) P with P[i, pi(i)] = 1, so the ground truth is X_GT = P.
* E is symmetric Gaussian noise placed on existing edges only (reading A15), zero diagonal.
* B ~ N(0, 1) (n x d); B'[pi(i)] = B[i] + N(0, sigma_B^2).
* Config 3 (n < n'): A' has n inliers (a noisy permuted copy of A) plus n'-n outliers whose
  every incident pair is an edge w.p. p with weight U(0,1) (reading A17); outlier attributes are
  independent N(0,1) and inlier attributes get N(0, 0.1^2) noise (reading A16).
* Seeds: config k uses base seed 1207_1114 + k with numpy PCG64; config 4's per-pair seeds come
  from SeedSequence(base).spawn(batch).

All arrays are float32 row-major (the GPU path's storage type); the oracle promotes to float64.
The paper's public datasets (CMU House, Oxford affine sets, Face 50, Stanford Bunny;
PAPER.md:463-636) are not in this container; these synthetic workloads stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

BASE_SEED = 1207_1114


@dataclass
class Problem:
    """One graph-matching instance plus the solver hyper-parameters it is run with.

    A (n x n), Ap (n' x n'), B (n x d) and Bp (n' x d) follow PAPER.md:135-141. lam, alpha,
    eps1, eps2, max_iter1 (I_0, outer) and max_iter2 (I_1, inner) follow PAPER.md:424-431.
    X0 is the initial soft assignment (None => 11^T/(n n')).
    perm[i] = planted partner of node i of G in G' (ground truth, -1 if none).
    """

    name: str
    A: np.ndarray
    Ap: np.ndarray
    B: Optional[np.ndarray]
    Bp: Optional[np.ndarray]
    lam: float
    alpha: float
    eps1: float
    eps2: float
    max_iter1: int
    max_iter2: int
    X0: Optional[np.ndarray] = None
    perm: Optional[np.ndarray] = None
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def n_prime(self) -> int:
        return self.Ap.shape[0]

    @property
    def d(self) -> int:
        return 0 if self.B is None else self.B.shape[1]


# --------------------------------------------------------------------------------------------
# graph primitives (sampling only)
# --------------------------------------------------------------------------------------------

def random_weighted_graph(rng: np.random.Generator, n: int, p: float) -> np.ndarray:
    """Symmetric n x n, zero diagonal; each upper pair an edge w.p. p with weight U(0,1)."""
    w = rng.random((n, n), dtype=np.float32)
    keep = rng.random((n, n), dtype=np.float32) < np.float32(p)
    up = np.triu(np.where(keep, w, np.float32(0.0)), k=1)
    return (up + up.T).astype(np.float32)


def edge_noise(rng: np.random.Generator, A: np.ndarray, sigma: float) -> np.ndarray:
    """Symmetric N(0, sigma^2) noise on the existing (nonzero) upper-triangle edges of A."""
    n = A.shape[0]
    if sigma == 0.0:
        return np.zeros_like(A)
    e = rng.standard_normal((n, n), dtype=np.float32) * np.float32(sigma)
    up = np.triu(np.where(A != 0, e, np.float32(0.0)), k=1)
    return (up + up.T).astype(np.float32)


def relabel(M: np.ndarray, pi: np.ndarray) -> np.ndarray:
    """Return M' with M'[pi(i), pi(j)] = M[i, j] (M' = P^T M P, P[i, pi(i)] = 1)."""
    inv = np.empty_like(pi)
    inv[pi] = np.arange(pi.size)
    return np.ascontiguousarray(M[np.ix_(inv, inv)])


def relabel_rows(M: np.ndarray, pi: np.ndarray) -> np.ndarray:
    """Return M' with M'[pi(i)] = M[i] (M' = P^T M)."""
    inv = np.empty_like(pi)
    inv[pi] = np.arange(pi.size)
    return np.ascontiguousarray(M[inv])


def planted_pair(rng, n, p, sigma_e, d=0, sigma_b=0.1):
    """(A, A', B, B', pi) for a planted isomorphic-with-noise pair of size n."""
    A = random_weighted_graph(rng, n, p)
    E = edge_noise(rng, A, sigma_e)
    pi = rng.permutation(n).astype(np.int64)
    Ap = relabel(A + E, pi)
    B = Bp = None
    if d > 0:
        B = rng.standard_normal((n, d), dtype=np.float32)
        noisy = B + rng.standard_normal((n, d), dtype=np.float32) * np.float32(sigma_b)
        Bp = relabel_rows(noisy, pi)
    return A, Ap, B, Bp, pi


# --------------------------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------------------------

def config1(seed: int = BASE_SEED + 1, n: int = 64) -> Problem:
    """BASELINE.json configs[0]: tiny planted isomorphism, n = n' = 64, p = 0.3, lambda = 0,
    X0 = 1/n * ones, alpha = 0.5, eps1 = eps2 = 1e-6, I0 = I1 = 100."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A, Ap, _, _, pi = planted_pair(rng, n, 0.3, 0.0)
    X0 = np.full((n, n), 1.0 / n, dtype=np.float32)
    return Problem("c1_tiny_planted", A, Ap, None, None, lam=0.0, alpha=0.5, eps1=1e-6,
                   eps2=1e-6, max_iter1=100, max_iter2=100, X0=X0, perm=pi, seed=seed)


def config2(seed: int = BASE_SEED + 2, n: int = 1000, d: int = 32) -> Problem:
    """BASELINE.json configs[1]: n = n' = 1000, p = 0.5, edge noise N(0, 0.05^2), d = 32,
    B' noise N(0, 0.1^2), lambda = 1, alpha = 0.5, eps = 1e-4, I0 = I1 = 300 (reading A8)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A, Ap, B, Bp, pi = planted_pair(rng, n, 0.5, 0.05, d=d, sigma_b=0.1)
    return Problem("c2_paper_scale", A, Ap, B, Bp, lam=1.0, alpha=0.5, eps1=1e-4, eps2=1e-4,
                   max_iter1=300, max_iter2=300, perm=pi, seed=seed)


def config3(seed: int = BASE_SEED + 3, n: int = 800, n_prime: int = 1000, d: int = 16) -> Problem:
    """BASELINE.json configs[2]: n = 800 < n' = 1000 with 200 outliers, p = 0.4, inlier noise
    N(0, 0.05^2), d = 16 (outlier attributes independent), lambda = 0.5, alpha = 0.5, eps = 1e-4."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = 0.4
    A = random_weighted_graph(rng, n, p)
    E = edge_noise(rng, A, 0.05)
    big = random_weighted_graph(rng, n_prime, p)   # supplies every pair touching an outlier
    big[:n, :n] = A + E                            # inlier block: noisy copy of A
    pi = rng.permutation(n_prime).astype(np.int64)
    Ap = relabel(big, pi)
    B = rng.standard_normal((n, d), dtype=np.float32)
    Bbig = rng.standard_normal((n_prime, d), dtype=np.float32)
    Bbig[:n] = B + rng.standard_normal((n, d), dtype=np.float32) * np.float32(0.1)
    Bp = relabel_rows(Bbig, pi)
    return Problem("c3_unequal_outliers", A, Ap, B, Bp, lam=0.5, alpha=0.5, eps1=1e-4, eps2=1e-4,
                   max_iter1=300, max_iter2=300, perm=pi[:n].copy(), seed=seed)


def config4(seed: int = BASE_SEED + 4, batch: int = 8192, n: int = 128, fixed: bool = True,
            first: int = 0, count: Optional[int] = None) -> list:
    """BASELINE.json configs[3]: `batch` independent pairs of n = n' = 128, p = 0.3, A' =
    P^T (A + N(0, 0.02^2) on edges) P per pair (per-pair seeds), lambda = 0. fixed=True is the
    fixed 20 x 20 throughput mode (eps = 0); fixed=False is eps = 1e-4, I = 100/100 (reading A8).
    `first`/`count` select a sub-range of pairs (same per-pair seeds as the full batch)."""
    children = np.random.SeedSequence(seed).spawn(batch)
    count = batch - first if count is None else count
    out = []
    for k in range(first, first + count):
        rng = np.random.Generator(np.random.PCG64(children[k]))
        A, Ap, _, _, pi = planted_pair(rng, n, 0.3, 0.02)
        if fixed:
            out.append(Problem(f"c4_pair{k}", A, Ap, None, None, lam=0.0, alpha=0.5, eps1=0.0,
                               eps2=0.0, max_iter1=20, max_iter2=20, perm=pi, seed=seed))
        else:
            out.append(Problem(f"c4_pair{k}", A, Ap, None, None, lam=0.0, alpha=0.5, eps1=1e-4,
                               eps2=1e-4, max_iter1=100, max_iter2=100, perm=pi, seed=seed))
    return out


def config5(seed: int = BASE_SEED + 5, n: int = 16384, d: int = 64) -> Problem:
    """BASELINE.json configs[4]: n = n' = 16384, p = 0.1 (dense storage), noise N(0, 0.05^2),
    d = 64 with N(0, 0.1^2) attribute noise, lambda = 1, alpha = 0.5, fixed 20 outer x 20 inner
    (eps = 0 => run exactly max_iter, reading A8). Smaller n keeps the same recipe."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A, Ap, B, Bp, pi = planted_pair(rng, n, 0.1, 0.05, d=d, sigma_b=0.1)
    return Problem("c5_large", A, Ap, B, Bp, lam=1.0, alpha=0.5, eps1=0.0, eps2=0.0,
                   max_iter1=20, max_iter2=20, perm=pi, seed=seed)


def random_problem(seed: int, n: int, n_prime: int, d: int = 0, p: float = 0.5, lam: float = 0.0,
                   alpha: float = 0.5, eps1: float = 1e-4, eps2: float = 1e-4, max_iter1: int = 50,
                   max_iter2: int = 50) -> Problem:
    """Small unrelated pair (no planted structure) for edge cases and ragged shapes."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = random_weighted_graph(rng, n, p)
    Ap = random_weighted_graph(rng, n_prime, p)
    B = Bp = None
    if d > 0:
        B = rng.standard_normal((n, d), dtype=np.float32)
        Bp = rng.standard_normal((n_prime, d), dtype=np.float32)
    return Problem(f"rand_{n}x{n_prime}_d{d}", A, Ap, B, Bp, lam=lam, alpha=alpha, eps1=eps1,
                   eps2=eps2, max_iter1=max_iter1, max_iter2=max_iter2, seed=seed)


def planted_unequal(seed: int, n: int, n_prime: int, d: int = 0, lam: float = 0.5,
                    eps1: float = 1e-5, eps2: float = 1e-5, max_iter1: int = 25,
                    max_iter2: int = 60) -> Problem:
    """Small config-3-style pair (planted noisy subgraph + outliers) of any orientation: when
    n > n' the roles of the two graphs are swapped (the larger graph carries the outliers)."""
    small, big = min(n, n_prime), max(n, n_prime)
    q = config3(seed=seed, n=small, n_prime=big, d=max(d, 1))
    B, Bp = (q.B, q.Bp) if d > 0 else (None, None)
    if n <= n_prime:
        A, Ap = q.A, q.Ap
    else:
        A, Ap, B, Bp = q.Ap, q.A, Bp, B
    return Problem(f"planted_{n}x{n_prime}_d{d}", A, Ap, B, Bp, lam=lam if d > 0 else 0.0,
                   alpha=0.5, eps1=eps1, eps2=eps2, max_iter1=max_iter1, max_iter2=max_iter2,
                   seed=seed)


def random_matrix(seed: int, rows: int, cols: int, scale: float = 1.0, shift: float = 0.0) -> np.ndarray:
    """Plain seeded float32 matrix (e.g. a Y for one projection sweep)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(scale)
            + np.float32(shift)).astype(np.float32)


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}


def stack_pairs(problems):
    """Pair-major dense arrays (A [b][n][n], A' [b][n'][n'], B, B') for the batched path."""
    A = np.ascontiguousarray(np.stack([p.A for p in problems]))
    Ap = np.ascontiguousarray(np.stack([p.Ap for p in problems]))
    B = Bp = None
    if problems[0].B is not None:
        B = np.ascontiguousarray(np.stack([p.B for p in problems]))
        Bp = np.ascontiguousarray(np.stack([p.Bp for p in problems]))
    return A, Ap, B, Bp


# --------------------------------------------------------------------------------------------
# fully connected Euclidean-distance graphs (the graph construction of the paper's
# real-data experiments E2-E4: "each edge represents Euclidean distance between two keypoints",
# PAPER.md:435; 128-d SIFT-like attributes with K_ij = inner products,
# P:527-532). Synthetic stand-in: no dataset item is reproduced.
# --------------------------------------------------------------------------------------------

def _rotation(rng, dim):
    Q, R = np.linalg.qr(rng.standard_normal((dim, dim)))
    Q = Q * np.sign(np.diag(R))
    if np.linalg.det(Q) < 0:
        Q[:, 0] = -Q[:, 0]
    return Q


def _unit_rows(M):
    M = np.abs(M)
    return (M / np.maximum(np.linalg.norm(M, axis=1, keepdims=True), 1e-12)).astype(np.float32)


def distance_pair(seed: int, n: int, n_outliers: int = 0, dim: int = 2, d: int = 128,
                  jitter: float = 0.01, attr_noise: float = 0.05, lam: float = 1.0,
                  alpha: float = 0.5, eps1: float = 1e-4, eps2: float = 1e-4, max_iter1: int = 300,
                  max_iter2: int = 300) -> Problem:
    """Points P in [0,1]^dim; the partner is a rigidly moved (rotation + translation), jittered,
    permuted copy plus `n_outliers` uniform outlier points. A_ij = ||p_i - p_j|| (fully connected,
    zero diagonal). Attributes: nonnegative unit 128-d vectors (SIFT-like), the
    partner's inlier attributes perturbed by `attr_noise` and re-normalised; K = B B'^T.
    n' = n + n_outliers >= n: slack rows (reading A1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    P = rng.random((n, dim))
    R = _rotation(rng, dim)
    Q_in = P @ R.T + rng.random(dim) + rng.standard_normal((n, dim)) * jitter
    lo, hi = Q_in.min(0), Q_in.max(0)
    Q_out = lo + rng.random((n_outliers, dim)) * (hi - lo)
    Q = np.vstack([Q_in, Q_out])
    npr = n + n_outliers
    pi = rng.permutation(npr).astype(np.int64)
    inv = np.empty_like(pi)
    inv[pi] = np.arange(npr)
    Qp = Q[inv]                                   # Q'[pi(i)] = Q[i]
    dist = lambda X: np.sqrt(np.maximum(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1), 0.0))
    A = dist(P).astype(np.float32)
    Ap = dist(Qp).astype(np.float32)
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(Ap, 0.0)
    A = ((A + A.T) / 2).astype(np.float32)
    Ap = ((Ap + Ap.T) / 2).astype(np.float32)
    B = _unit_rows(rng.random((n, d)))
    Bq = np.vstack([_unit_rows(B + rng.standard_normal((n, d)) * attr_noise),
                    _unit_rows(rng.random((n_outliers, d)))])
    Bp = np.ascontiguousarray(Bq[inv])
    return Problem(f"dist{dim}d_{n}+{n_outliers}", A, Ap, B, Bp, lam=lam, alpha=alpha, eps1=eps1,
                   eps2=eps2, max_iter1=max_iter1, max_iter2=max_iter2, perm=pi[:n].copy(), seed=seed,
                   meta={"dim": dim, "jitter": jitter, "attr_noise": attr_noise})


def ga_pair(seed: int, n: int, n_prime: Optional[int] = None, p: float = 0.3, sigma_e: float = 0.02,
            d: int = 0, lam: float = 0.0, q: float = 8.0, eps1: float = 1e-6, eps2: float = 1e-6,
            max_iter1: int = 100, max_iter2: int = 100) -> Problem:
    """FastGA workload: a planted noisy pair (config-1/2 recipe; when
    n != n' the config-3 outlier recipe) whose edge weights are multiplied by
    s = sqrt(q / (p n / 3)), so that the expected sum_j A_ij^2 is q whatever n is. GA's exponent
    beta (A X A')_ia then peaks near beta_max * q at a permutation (about 80 with the defaults),
    which keeps exp's argument well conditioned for an fp32 product. Sampling/scaling only."""
    n_prime = n if n_prime is None else n_prime
    if n_prime == n:
        rng = np.random.Generator(np.random.PCG64(seed))
        A, Ap, B, Bp, pi = planted_pair(rng, n, p, sigma_e, d=d, sigma_b=0.1)
    else:
        base = planted_unequal(seed, n, n_prime, d=d, lam=lam)
        A, Ap, B, Bp, pi = base.A, base.Ap, base.B, base.Bp, None
    s = np.float32(np.sqrt(q / (p * max(n, n_prime) / 3.0)))
    A = (A * s).astype(np.float32)
    Ap = (Ap * s).astype(np.float32)
    return Problem(f"ga_{n}x{n_prime}_d{d}", A, Ap, B, Bp, lam=lam if d > 0 else 0.0, alpha=0.0,
                   eps1=eps1, eps2=eps2, max_iter1=max_iter1, max_iter2=max_iter2, perm=pi,
                   seed=seed, meta={"weight_scale": float(s)})
