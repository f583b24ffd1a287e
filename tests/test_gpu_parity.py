"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): max|X_gpu - X_oracle| <= 1e-4 after each of the first 10
outer iterations and at termination; objective relative difference <= 1e-4; >= 99% identical
assignments (identical on planted cases). Bit-exact where the paper's worked values are dyadic.
"""
import json
import os

import numpy as np
import pytest

from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs

from .parity import X_TOL, assert_parity, run_pair

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1207_1114_b200 as F
    F.lib()   # loud failure if the library is missing (no fallback)


PRECS = [pytest.param(0, id="tf32x3"), pytest.param(2, id="simt"),
         pytest.param(3, id="int8ozaki")]  # PREC_TF32X3, PREC_FP32_SIMT, PREC_INT8_OZAKI


# ---------------------------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------------------------

def test_dyadic_sweep_bit_exact(golden_dir):
    import paper_1207_1114_b200 as F
    g = json.load(open(os.path.join(golden_dir, "dyadic_sweep.json")))
    for c in g["cases"]:
        Y = torch.tensor(g["Y0"], dtype=torch.float32, device="cuda")
        s, d = F.project(Y, c["eps2"], c["max_iter2"])
        assert s == c["sweeps"] and d == c["delta"]
        assert torch.equal(Y.cpu(), torch.diag(torch.tensor([c["diag"]] * 2)))


@pytest.mark.parametrize("m", [1, 2, 37, 300, 513, 1000, 1500])
def test_sweeps_vs_oracle(m):
    import paper_1207_1114_b200 as F
    Y0 = inputs.random_matrix(1000 + m, m, m, scale=3.0, shift=0.2)
    for k in (1, 7):
        Y = torch.from_numpy(Y0).cuda()
        s, d = F.project(Y, 0.0, k)
        Yo, so, do = O.project_loop(Y0.astype(np.float64), 0.0, k)
        assert s == so == k
        err = np.max(np.abs(Y.cpu().numpy().astype(np.float64) - Yo))
        assert err <= 2e-6 * max(1.0, np.max(np.abs(Y0))), err
        assert abs(d - do) <= 2e-6 * max(1.0, np.max(np.abs(Y0)))


@pytest.mark.parametrize("m,stop", [(300, 6), (513, 4), (2100, 8), (700, 3)])
def test_eps2_stop_between_checkpoints(m, stop):
    # the streaming kernel stores Y only after every other sweep (checkpointed sweeps):
    # an eps2 stop after an even sweep takes one more pass to store that sweep's Y. eps2 is
    # placed between the oracle's delta of sweep `stop` and the smallest delta before it.
    import paper_1207_1114_b200 as F
    Y0 = inputs.random_matrix(2000 + m, m, m, scale=3.0, shift=0.2)
    Yo = Y0.astype(np.float64)
    deltas = []
    for _ in range(stop):
        Yo, d = O.sweep(Yo)
        deltas.append(d)
    lo, hi = deltas[-1], min(deltas[:-1])
    assert lo < hi / 1.05, deltas          # a margin the fp32 deltas cannot cross
    eps2 = float(np.sqrt(lo * hi))
    Y = torch.from_numpy(Y0).cuda()
    s, d = F.project(Y, eps2, 100)
    assert s == stop
    scale = max(1.0, np.max(np.abs(Y0)))
    assert np.max(np.abs(Y.cpu().numpy().astype(np.float64) - Yo)) <= 2e-6 * scale
    assert abs(d - deltas[-1]) <= 2e-6 * scale


GEMM_VARIANTS = [pytest.param(0, 2, id="tf32x3-cg2"), pytest.param(0, 1, id="tf32x3-cg1"),
                 pytest.param(2, 2, id="simt")]


@pytest.mark.parametrize("prec,cg", GEMM_VARIANTS)
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (129, 257, 33), (300, 1000, 700),
                                   (1000, 1000, 1000), (256, 512, 4096), (1500, 700, 2048)])
def test_gemm_nt_error_bound(prec, cg, M, N, K):
    import paper_1207_1114_b200 as F
    r = np.random.default_rng(M * 7 + N * 3 + K)
    P = r.random((M, K), dtype=np.float32) * (r.random((M, K)) < 0.5)
    Q = r.random((N, K), dtype=np.float32)
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    F.gemm_nt(torch.from_numpy(P.astype(np.float32)).cuda(), torch.from_numpy(Q).cuda(), C, prec, cg)
    exact = P.astype(np.float64) @ Q.astype(np.float64).T
    mag = np.abs(P.astype(np.float64)) @ np.abs(Q.astype(np.float64)).T
    # fp32 accumulation: |err| <= K u |P||Q|^T (u = 2^-24); 3xTF32 adds <= 3 * 2^-22 |P||Q|^T
    bound = (K * 2.0**-24 + 3 * 2.0**-22) * mag + 1e-30
    err = np.abs(C.cpu().numpy().astype(np.float64) - exact)
    assert np.all(err <= bound), float(np.max(err / bound))


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (129, 257, 33), (300, 1000, 700),
                                   (1000, 1000, 1000), (256, 512, 4096), (1500, 700, 2048),
                                   (640, 384, 16384), (2500, 2100, 96)])   # last: 170 tiles, ragged
@pytest.mark.parametrize("signed", [False, True])
def test_gemm_nt_int8_ozaki_error_bound(M, N, K, signed):
    # Ozaki int8 (PRECISION = 3): rows = 2^e * (3 signed 7-bit digits), digit pairs p + q <= 4
    # exact in int32. Per element: representation error <= 2^-21 of the row scale per operand entry,
    # dropped pairs (p + q >= 5, remainder digits |d| <= 64) <= 2^-22 s_P s_Q per k, fp32 combine
    # <= 2^-22 |P||Q|^T
    import paper_1207_1114_b200 as F
    r = np.random.default_rng(M * 5 + N * 11 + K + signed)
    P = (r.random((M, K)) * (r.random((M, K)) < 0.5)).astype(np.float32)
    Q = r.random((N, K)).astype(np.float32) * np.float32(1e-3)
    if signed:
        P = (P - np.float32(0.25) * (P > 0)).astype(np.float32)
        Q = (Q * np.where(r.random((N, K)) < 0.5, -1, 1)).astype(np.float32)
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    F.gemm_nt(torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda(), C, F.PREC_INT8_OZAKI, 2)
    P64, Q64 = P.astype(np.float64), Q.astype(np.float64)
    exact = P64 @ Q64.T
    scale = lambda M_: np.exp2(np.floor(np.log2(np.maximum(np.max(np.abs(M_), 1), 1e-300))) + 1)
    sP, sQ = scale(P64), scale(Q64)
    rep = 2.0**-21 * (np.abs(P64).sum(1)[:, None] * sQ[None, :] + sP[:, None] * np.abs(Q64).sum(1)[None, :])
    bound = rep + K * 2.0**-22 * sP[:, None] * sQ[None, :] + 2.0**-22 * (np.abs(P64) @ np.abs(Q64).T) + 1e-30
    err = np.abs(C.cpu().numpy().astype(np.float64) - exact)
    assert np.all(err <= bound), float(np.max(err / bound))
    # and it is far more accurate than 1xTF32 (2^-11) on these inputs
    assert np.max(err / (np.abs(P64) @ np.abs(Q64).T + 1e-30)) < 2.0**-16


# ---------------------------------------------------------------------------------------------
# Algorithm 1 end to end
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("pk", [pytest.param(0, id="auto-onchip"), pytest.param(1, id="streaming")])
def test_dyadic_two_node_bit_exact(golden_dir, prec, pk):
    import paper_1207_1114_b200 as F
    g = json.load(open(os.path.join(golden_dir, "dyadic_two_node.json")))
    s = F.Solver(2, 2, 1)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_option(F.OPT_PROJ_KERNEL, pk)
    arr = lambda k: np.array(g[k], np.float32)
    s.set_graphs(arr("A"), arr("Ap"), arr("B"), arr("Bp"))
    s.set_x0(arr("X0"))
    for it in g["iters"]:
        X, rep = s.iterate(g["alpha"], g["lam"], 0.0, g["eps2"], 1, g["max_iter2"])
        assert rep.sweeps == [it["sweeps"]]
        assert rep.mu[0] == pytest.approx(it["mu"], rel=1e-7)
        if "X_rtol" in it:
            assert np.allclose(X, it["X"], rtol=1e-6, atol=0)
        else:
            assert np.array_equal(X, np.array(it["X"], np.float32)) and rep.rho == [it["rho"]]
    assert list(s.discretize()) == g["assignment"]


@pytest.mark.parametrize("prec", PRECS)
def test_config1_planted(prec):
    p = inputs.config1()
    res = run_pair(p, prec)
    assert_parity(res, planted=p.perm)
    assert np.array_equal(res.assign_gpu, p.perm)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", [(37, 53, 3), (53, 37, 3), (1, 1, 0), (1, 5, 2), (130, 129, 4),
                                   (60, 40, 4), (600, 520, 8)])
@pytest.mark.parametrize("slack_mode", [0, 1])
@pytest.mark.parametrize("pk", [pytest.param(0, id="auto-onchip"), pytest.param(1, id="streaming")])
def test_ragged_planted_pairs(prec, shape, slack_mode, pk):
    # planted noisy subgraph pairs of both orientations (slack rows / slack columns, reading A1)
    n, npr, d = shape
    p = inputs.planted_unequal(17 + n + npr, n, npr, d=d)
    res = run_pair(p, prec, slack_mode=slack_mode, proj_kernel=pk)
    assert_parity(res)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", [(37, 53, 3), (53, 37, 0), (130, 129, 4), (515, 1029, 2)])
def test_ragged_random_pairs_short(prec, shape):
    # unrelated random pairs: no planted optimum, so long runs can be chaotic (the fp32 twin drifts
    # by ~2e-4 after 15 iterations on (53, 37)); parity is asserted over the first 6 iterations,
    # where the twin's drift is < 2e-5.
    n, npr, d = shape
    p = inputs.random_problem(17 + n + npr, n, npr, d=d, lam=0.7, eps1=1e-5, eps2=1e-5,
                              max_iter1=6, max_iter2=60)
    res = run_pair(p, prec, lockstep=6)
    assert max(res.lockstep_max) <= 1e-4 and res.final_diff <= 1e-4


@pytest.mark.parametrize("prec", PRECS)
def test_rescale_off(prec):
    p = inputs.random_problem(99, 40, 30, d=2, lam=0.5, eps1=0.0, eps2=1e-6, max_iter1=8,
                              max_iter2=50)
    res = run_pair(p, prec, rescale=0)
    assert max(res.lockstep_max) <= 1e-4 and res.final_diff <= 1e-4


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("pk", [pytest.param(0, id="auto-onchip"), pytest.param(1, id="streaming")])
def test_config2_paper_scale(prec, pk):
    p = inputs.config2()
    res = run_pair(p, prec, proj_kernel=pk)
    assert_parity(res, planted=p.perm)
    assert np.mean(res.assign_gpu == p.perm) >= 0.99


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("pk", [pytest.param(0, id="auto-onchip"), pytest.param(1, id="streaming")])
def test_config3_unequal_outliers(prec, pk):
    p = inputs.config3()
    res = run_pair(p, prec, proj_kernel=pk)
    assert_parity(res)


@pytest.mark.parametrize("prec,cg", [pytest.param(0, 2, id="tf32x3"), pytest.param(0, 1, id="tf32x3-cg1"),
                                     pytest.param(2, 2, id="simt"), pytest.param(3, 2, id="int8ozaki")])
def test_config5_recipe_reduced(prec, cg):
    # the c5 recipe (p = 0.1, d = 64, lambda = 1, fixed 20 x 20) at n = 2048: spans 8 x 8 pair tiles
    # of the GEMM and 4 x 16 projection tile columns, exercised by the oracle in seconds
    p = inputs.config5(n=2048)
    p.max_iter1 = 6
    res = run_pair(p, prec, lockstep=6, cta_group=cg)
    assert max(res.lockstep_max) <= 1e-4 and res.final_diff <= 1e-4
    assert res.gpu_sweeps == res.oracle_sweeps == [20] * 6


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
def test_config5_recipe_ragged_many_tiles(prec):
    # n = 2600: 11 x 21 = 231 GEMM pair tiles (> 74 CTA pairs, so CTAs run several tiles and the
    # int8 epilogue's register path runs as well as its staged last tile), ragged in M (40 rows) and
    # N (40 columns), with the lambda K epilogue (d = 64); ragged projection tiles (2600 = 5 x 512 + 40)
    p = inputs.config5(n=2600)
    p.max_iter1 = 3
    res = run_pair(p, prec, lockstep=3, proj_kernel=1)
    assert max(res.lockstep_max) <= 1e-4 and res.final_diff <= 1e-4
    assert res.gpu_sweeps == res.oracle_sweeps == [20] * 3


# ---------------------------------------------------------------------------------------------
# contract details
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cg", [1, 2])
def test_tf32_single_pass_error_is_tf32_sized(cg):
    # plain 1xTF32 (reported separately, not parity-accurate): error ~ 2^-11 relative per operand
    import paper_1207_1114_b200 as F
    r = np.random.default_rng(3)
    M, N, K = 384, 640, 1024
    P = r.random((M, K), dtype=np.float32); Q = r.random((N, K), dtype=np.float32)
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    F.gemm_nt(torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda(), C, F.PREC_TF32, cg)
    exact = P.astype(np.float64) @ Q.astype(np.float64).T
    rel = np.max(np.abs(C.cpu().numpy() - exact) / exact)
    assert 1e-7 < rel < 2.0**-9


def test_k_single_steps_equal_one_call_bitwise():
    import paper_1207_1114_b200 as F
    p = inputs.random_problem(5, 64, 48, d=4, lam=0.5, eps1=0.0, eps2=1e-6, max_iter1=6, max_iter2=40)
    a = F.Solver(64, 48, 4); a.set_graphs(p.A, p.Ap, p.B, p.Bp)
    Xa, _ = a.iterate(p.alpha, p.lam, 0.0, p.eps2, 6, p.max_iter2)
    b = F.Solver(64, 48, 4); b.set_graphs(p.A, p.Ap, p.B, p.Bp)
    for _ in range(6):
        Xb, _ = b.iterate(p.alpha, p.lam, 0.0, p.eps2, 1, p.max_iter2)
    assert np.array_equal(Xa, Xb)


def test_check_every_does_not_change_result():
    import paper_1207_1114_b200 as F
    p = inputs.config1()
    outs = []
    for ce in (1, 3, 64):
        s = F.Solver(p.n, p.n_prime, 0)
        s.set_option(F.OPT_CHECK_EVERY, ce)
        s.set_graphs(p.A, p.Ap); s.set_x0(p.X0)
        X, rep = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, p.max_iter1, p.max_iter2)
        outs.append((X, rep.iterations, rep.sweeps))
    for X, it, sw in outs[1:]:
        assert np.array_equal(X, outs[0][0]) and it == outs[0][1] and sw == outs[0][2]


def test_errors():
    import paper_1207_1114_b200 as F
    s = F.Solver(4, 3, 0)
    with pytest.raises(F.FastPFPError) as e:
        s.iterate(0.5, 0.0, 1e-4, 1e-4, 1, 1)
    assert e.value.status == F.ESTATE
    A = np.eye(4, dtype=np.float32); A[0, 1] = 1.0
    with pytest.raises(F.FastPFPError) as e:
        s.set_graphs(A, np.eye(3, dtype=np.float32))
    assert e.value.status == F.ESYM
    A = np.eye(4, dtype=np.float32); A[2, 2] = np.nan
    with pytest.raises(F.FastPFPError) as e:
        s.set_graphs(A, np.eye(3, dtype=np.float32))
    assert e.value.status == F.ENONFINITE
    s.set_graphs(np.eye(4, dtype=np.float32), np.eye(3, dtype=np.float32))
    with pytest.raises(F.FastPFPError) as e:
        s.iterate(1.5, 0.0, 1e-4, 1e-4, 1, 1)
    assert e.value.status == F.EINVAL
    X, rep = s.iterate(0.5, 0.0, 1e-4, 1e-4, 3, 5)
    assert rep.iterations >= 1


def test_device_inputs_match_host_inputs():
    import paper_1207_1114_b200 as F
    p = inputs.random_problem(8, 50, 70, d=3, lam=1.0, eps1=0.0, eps2=1e-6, max_iter1=4, max_iter2=30)
    a = F.Solver(50, 70, 3); a.set_graphs(p.A, p.Ap, p.B, p.Bp)
    b = F.Solver(50, 70, 3)
    b.set_graphs(*(torch.from_numpy(x).cuda() for x in (p.A, p.Ap, p.B, p.Bp)))
    Xa, _ = a.iterate(p.alpha, p.lam, 0.0, p.eps2, 4, p.max_iter2)
    Xb, _ = b.iterate(p.alpha, p.lam, 0.0, p.eps2, 4, p.max_iter2)
    assert np.array_equal(Xa, Xb)
    out = torch.empty((50, 70), dtype=torch.float32, device="cuda")
    b.copy_x(out)
    assert np.array_equal(out.cpu().numpy(), Xb)


@pytest.mark.parametrize("shape", [(300, 200), (200, 300), (1000, 1000), (1, 9), (9, 1), (777, 513)])
@pytest.mark.parametrize("kind", ["ties", "noisy_perm", "constant"])
def test_gpu_greedy_equals_sequential_greedy(shape, kind):
    # GPU locally-dominant rounds (+ host finish for tie chains) == Steps 1-3 of P:372-379
    import paper_1207_1114_b200 as F
    n, npr = shape
    r = np.random.default_rng(n * 31 + npr)
    if kind == "ties":
        X = (np.round(r.random((n, npr)) * 7) / 7).astype(np.float32)
    elif kind == "noisy_perm":
        X = (r.random((n, npr)) * 0.1).astype(np.float32)
        k = min(n, npr)
        X[r.permutation(n)[:k], r.permutation(npr)[:k]] += 1.0
    else:
        X = np.full((n, npr), 0.25, np.float32)
    s = F.Solver(n, npr, 0)
    s.set_graphs(np.zeros((n, n), np.float32), np.zeros((npr, npr), np.float32))
    s.set_x0(X)
    a = s.discretize()
    assert np.array_equal(a, O.greedy_discretize(X.astype(np.float64)))


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("dims", [(392, 0, 3), (500, 40, 2)])
def test_distance_workload_parity(prec, dims):
    # fully connected Euclidean-distance graphs + 128-d attributes (E2-E4 style)
    n, outl, dim = dims
    p = inputs.distance_pair(21 + n, n, n_outliers=outl, dim=dim, jitter=0.005, lam=10.0,
                             max_iter1=60, max_iter2=300)
    res = run_pair(p, prec)
    assert_parity(res)
    assert np.mean(res.assign_gpu == p.perm) >= 0.95


@pytest.mark.parametrize("shape", [(129, 129, 2), (700, 333, 4), (1400, 1500, 4), (2200, 2100, 4)])
def test_onchip_tilings_lockstep(shape):
    # the on-chip projection forced (OPT_PROJ_KERNEL = 2) over tilings the configs do not reach:
    # m = 129 (the first multi-tile size: 5 x 5 tiles), m = 700 with slack columns, m = 1500 (12 x 12
    # tiles of 125 x 128, 4 column chunks per lane), m = 2200 (184 x 184 tiles, 6 column chunks per
    # lane, near the shared-memory limit of the fp32 tile). The tagged
    # exchange of partial sums runs every sweep; lockstep parity with the oracle after each of the
    # first 3 outer iterations (eps1 = 0, 40 sweeps cap: the tiles exchange 40 times per iteration).
    n, npr, d = shape
    p = inputs.planted_unequal(300 + n, n, npr, d=d, eps1=0.0, eps2=1e-7, max_iter1=3, max_iter2=40)
    res = run_pair(p, 3, lockstep=3, proj_kernel=2)
    assert max(res.lockstep_max) <= X_TOL, res.lockstep_max
    assert all(abs(a - b) <= 1 for a, b in zip(res.gpu_sweeps, res.oracle_sweeps)), (res.gpu_sweeps, res.oracle_sweeps)
