"""Parity at BASELINE.json's full c5 size (n = n' = 16384, d = 64), in the launch configuration
bench.py times (int8 Ozaki GEMMs, streaming bulk-ring projection, 20 sweeps), on sampled outputs
the fp64 oracle's formulas compute one by one, plus properties that hold at any size.

* One outer iteration with I1 = 1 from a random X0: for sampled rows i the exact fp64 values of
  G = A X0 A' + lambda K and of the first sweep Z = max(G + (1 + sigma/m - r_i - c_j)/m, 0)
   need only A[i,:] X0 A', the column sums c = (1^T A) X0 A' + lambda 1^T K and
  sigma = 1^T c — O(n^2) each, seconds in numpy. The GPU's Y rows must match within the GEMM's
  error bound; X1 must equal ((1 - alpha) X0 + alpha Z) / mu on the sampled rows.
* The bench configuration (I1 = 20, two outer iterations): X >= 0, max X = 1 (rescale), and the
  smaller-side-sum recursion s_{t+1} = ((1 - alpha) s_t + alpha r(Z_t)) / mu_t of DESIGN.md §4 on
  every row (r(Z_t) from the GPU's own projection output, fastpfp_copy_y).
These use the oracle's formulas (oracle/fastpfp.py) written for single rows; nothing here comes
from the CUDA path except the values under test.
"""
import numpy as np
import pytest

from paper_1207_1114_b200 import inputs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROWS = [0, 1, 4097, 8191, 12288, 16383]


@pytest.fixture(scope="module")
def c5():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1207_1114_b200 as F
    F.lib()
    return inputs.config5()


def _solver(p):
    import paper_1207_1114_b200 as F
    s = F.Solver(p.n, p.n_prime, p.d)
    s.set_option(F.OPT_PRECISION, F.PREC_INT8_OZAKI)   # bench.py's default
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    return s


def test_c5_full_size_first_sweep_sampled_rows(c5):
    p = c5
    n, m = p.n, p.n
    X0 = inputs.random_matrix(91, n, n, scale=1.0, shift=0.0)
    X0 = (np.abs(X0) / np.float32(n)).astype(np.float32)           # nonnegative, O(1/n)
    s = _solver(p)
    s.set_x0(X0)
    X1, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 1)
    Y = s.copy_y()
    s.close()
    A = p.A.astype(np.float64); Ap = p.Ap.astype(np.float64); X = X0.astype(np.float64)
    B = p.B.astype(np.float64); Bp = p.Bp.astype(np.float64)
    # column sums of G = A X A' + lambda K and sigma (fp64, O(n^2))
    c = ((A.sum(0) @ X) @ Ap) + p.lam * (B.sum(0) @ Bp.T)
    sigma = c.sum()
    cM = ((np.abs(A).sum(0) @ X) @ np.abs(Ap)) + p.lam * (np.abs(B).sum(0) @ np.abs(Bp).T)
    for i in ROWS:
        Gi = (A[i] @ X) @ Ap + p.lam * (B[i] @ Bp.T)                 # row i of the gradient
        Mi = (np.abs(A[i]) @ X) @ np.abs(Ap) + p.lam * np.abs(B[i]) @ np.abs(Bp.T)
        ri = Gi.sum()
        Zi = np.maximum(Gi + (1.0 + sigma / m - ri - c) / m, 0.0)  # P1 then P2, one sweep
        # GPU G: fp32 storage (2^-24 |G|) + the int8 GEMM (<= 2^-21 |A||X||A'|); the sums r_i, c_j,
        # sigma of that G carry the summed element errors into the correction (/m, /m^2)
        tol = (2.0**-20 * (Mi + np.abs(Gi)) + 2.0**-20 * (Mi.sum() + cM) / m
               + 2.0**-20 * cM.sum() / m**2 + 1e-12)
        err = np.abs(Y[i].astype(np.float64) - Zi)
        assert np.all(err <= tol), (i, float(np.max(err / tol)))
        # Algorithm 1 lines 8-9 on the GPU's own Z: X1 = ((1 - alpha) X0 + alpha Z) / mu
        Xt = (1 - p.alpha) * X[i] + p.alpha * Y[i].astype(np.float64)
        ref = (Xt / rep.mu[0]).astype(np.float32)
        assert np.all(np.abs(X1[i] - ref) <= np.spacing(ref))      # fp64 fma vs mul+add: <= 1 ulp
    assert float(X1.max()) == 1.0 and float(X1.min()) >= 0.0


def test_c5_full_size_bench_configuration_properties(c5):
    p = c5
    s = _solver(p)
    X_prev = np.full((p.n, p.n_prime), 1.0 / (p.n * p.n_prime), np.float64)
    for t in range(2):
        X, rep = s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, p.max_iter2)
        Z = s.copy_y().astype(np.float64)
        assert rep.sweeps == [20]
        assert float(X.max()) == 1.0 and float(X.min()) >= 0.0
        # smaller-side sums (rows, n = n'): s_{t+1} = ((1 - alpha) s_t + alpha r(Z_t)) / mu_t
        lhs = X.astype(np.float64).sum(1)
        rhs = ((1 - p.alpha) * X_prev.sum(1) + p.alpha * Z.sum(1)) / rep.mu[0]
        assert np.max(np.abs(lhs - rhs)) <= 1e-6 * max(1.0, float(np.max(np.abs(rhs))))
        # P2 leaves the projection output nonnegative (20 sweeps are far from the doubly stochastic
        # limit at this size: column sums are still O(10^3) after the first outer iteration)
        assert Z.min() >= 0.0
        X_prev = X.astype(np.float64)
    a = s.discretize()
    s.close()
    assert np.array_equal(np.sort(a), np.arange(p.n))        # greedy on n = n': a permutation
