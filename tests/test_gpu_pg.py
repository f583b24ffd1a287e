"""GPU parity of the Projected Gradient variant {pg} against the oracle."""
import json
import os

import numpy as np
import pytest

from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs

from .parity import run_pair

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

PRECS = [pytest.param(0, id="tf32x3"), pytest.param(2, id="simt"), pytest.param(3, id="int8ozaki")]
PKS = [pytest.param(0, id="auto"), pytest.param(1, id="streaming")]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1207_1114_b200 as F
    F.lib()


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("pk", PKS)
def test_pg_dyadic_bit_exact(golden_dir, prec, pk):
    import paper_1207_1114_b200 as F
    g = json.load(open(os.path.join(golden_dir, "dyadic_pg.json")))
    s = F.Solver(2, 2, 1)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_option(F.OPT_PROJ_KERNEL, pk)
    s.set_option(F.OPT_METHOD, F.METHOD_PG)
    arr = lambda k: np.array(g[k], np.float32)
    s.set_graphs(arr("A"), arr("Ap"), arr("B"), arr("Bp"))
    s.set_x0(arr("X0"))
    for it in g["iters"]:
        X, rep = s.iterate(g["alpha"], g["lam"], 0.0, g["eps2"], 1, g["max_iter2"])
        assert np.array_equal(X, np.array(it["X"], np.float32))
        assert rep.sweeps == [it["sweeps"]] and rep.rho == [it["rho"]]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("pk", PKS)
@pytest.mark.parametrize("shape", [(64, 64, 0), (200, 160, 4), (160, 200, 4)])
def test_pg_lockstep_vs_oracle(prec, pk, shape):
    n, npr, d = shape
    p = inputs.planted_unequal(5 + n, n, npr, d=d, eps1=1e-6, eps2=1e-6, max_iter1=12, max_iter2=200)
    p.alpha = 0.01
    res = run_pair(p, prec, lockstep=12, proj_kernel=pk, method=1)
    assert max(res.lockstep_max) <= 1e-4, res.lockstep_max
    assert res.final_diff <= 1e-4


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
def test_pg_many_ragged_tiles(prec):
    # n = 2600 (231 ragged GEMM pair tiles): the PG epilogue (X + alpha (A X A' + lambda K)) on the
    # int8 kernel's register path as well as its staged last tile; streaming projection
    p = inputs.config5(n=2600)
    p.alpha = 0.01
    p.max_iter1 = 2
    p.max_iter2 = 10
    res = run_pair(p, prec, lockstep=2, proj_kernel=1, method=1)
    assert max(res.lockstep_max) <= 1e-4, res.lockstep_max
    assert res.final_diff <= 1e-4


def test_pg_dist_world1():
    import paper_1207_1114_b200 as F
    p = inputs.config5(n=1024, d=8)
    uid = F.nccl_unique_id()
    s = F.Solver(p.n, p.n_prime, p.d, dist=(0, 1, uid))
    s.set_option(F.OPT_METHOD, F.METHOD_PG)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, method="pg")
    for _ in range(4):
        X, _ = s.iterate(0.01, p.lam, 0.0, 0.0, 1, 20)
        Xo, _ = st.iterate(p.lam, 0.01, 0.0, 0.0, 1, 20)
        assert np.max(np.abs(X.astype(np.float64) - Xo)) <= 1e-4
