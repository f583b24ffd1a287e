"""GPU tests of the row-sharded path (fastpfp_create_dist) at world size 1: the NCCL collectives
(1-rank communicator), the 3-D TMA K-loop over gathered U blocks and the phase-split projection
kernels all run; results must match the unsharded path and the fp64 oracle. (Multi-GPU runs use the
same code with world > 1; the decomposition itself is checked with 2 gloo ranks on CPU.)"""
import numpy as np
import pytest

from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs

from .parity import X_TOL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1207_1114_b200 as F
    F.lib()


def _dist_solver(p):
    import paper_1207_1114_b200 as F
    uid = F.nccl_unique_id()
    return F.Solver(p.n, p.n_prime, p.d, dist=(0, 1, uid))


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
def test_dist_world1_matches_single_and_oracle(prec):
    import paper_1207_1114_b200 as F
    p = inputs.config5(n=2048)
    a = F.Solver(p.n, p.n_prime, p.d)
    a.set_option(F.OPT_PRECISION, prec)
    a.set_graphs(p.A, p.Ap, p.B, p.Bp)
    b = _dist_solver(p)
    b.set_option(F.OPT_PRECISION, prec)
    b.set_graphs(p.A, p.Ap, p.B, p.Bp)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp)
    for t in range(4):
        Xa, ra = a.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 20)
        Xb, rb = b.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 20)
        Xo, _ = st.iterate(p.lam, p.alpha, 0.0, 0.0, 1, 20)
        assert rb.sweeps == [20]
        assert np.max(np.abs(Xa - Xb)) <= 1e-6
        assert np.max(np.abs(Xb.astype(np.float64) - Xo)) <= X_TOL
    fo = O.objective(st.A, st.Ap, st.K, st.X, p.lam)
    assert abs(b.objective(p.lam) - fo) <= 1e-4 * abs(fo)
    assert np.array_equal(b.discretize(), O.greedy_discretize(st.X))


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
@pytest.mark.parametrize("slack_mode", [0, 1])
def test_dist_world1_slack_columns(slack_mode, prec):
    import paper_1207_1114_b200 as F
    p = inputs.planted_unequal(77, 1024, 900, d=4, eps1=1e-5, eps2=1e-5, max_iter1=8, max_iter2=60)
    s = _dist_solver(p)
    s.set_option(F.OPT_SLACK_MODE, slack_mode)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, slack_mode="reset" if slack_mode else "persist")
    for t in range(5):
        X, r = s.iterate(p.alpha, p.lam, p.eps1, p.eps2, 1, p.max_iter2)
        Xo, ro = st.iterate(p.lam, p.alpha, p.eps1, p.eps2, 1, p.max_iter2)
        assert np.max(np.abs(X.astype(np.float64) - Xo)) <= X_TOL
        assert abs(r.sweeps[0] - ro.sweeps[0]) <= 1


def test_dist_rejects_unsupported_shapes():
    import paper_1207_1114_b200 as F
    uid = F.nccl_unique_id()
    with pytest.raises(F.FastPFPError):
        F.Solver(800, 1000, 0, dist=(0, 1, uid))     # n < n'
    with pytest.raises(F.FastPFPError):
        F.Solver(1000, 1000, 0, dist=(0, 1, uid))    # n/P not a multiple of 32
    s = F.Solver(96, 96, 0, dist=(0, 1, uid))        # n/P = 96: fine for TF32, not for int8
    with pytest.raises(F.FastPFPError):
        s.set_option(F.OPT_PRECISION, F.PREC_INT8_OZAKI)
    s.close()


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
@pytest.mark.parametrize("blocks,M,N,kb", [(2, 300, 520, 256), (4, 256, 384, 128), (8, 513, 129, 256)])
def test_blocked_k_loop_gemm_matches_dense(prec, blocks, M, N, kb):
    # the 3-D TMA K-loop over [P][N][K/P] rank blocks that GEMM2 of a P-rank run uses (it only runs
    # when P > 1): same product as the dense GEMM, within the same error bound
    import paper_1207_1114_b200 as F
    K = blocks * kb
    r = np.random.default_rng(blocks * 1000 + M)
    P = (r.random((M, K)) * (r.random((M, K)) < 0.5)).astype(np.float32)
    Q = r.random((N, K)).astype(np.float32)
    Cb = torch.empty((M, N), dtype=torch.float32, device="cuda")
    Cd = torch.empty((M, N), dtype=torch.float32, device="cuda")
    F.gemm_nt_blocked(torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda(), Cb, blocks, prec)
    F.gemm_nt(torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda(), Cd, prec, 2)
    exact = P.astype(np.float64) @ Q.astype(np.float64).T
    mag = np.abs(P.astype(np.float64)) @ np.abs(Q.astype(np.float64)).T
    err_b = np.abs(Cb.cpu().numpy().astype(np.float64) - exact)
    assert np.all(err_b <= (K * 2.0**-24 + 4 * 2.0**-21) * mag + 1e-30), float(np.max(err_b / (mag + 1e-30)))
    if prec == 3:   # same digits, same per-class integer sums: identical to the dense int8 product
        assert np.array_equal(Cb.cpu().numpy(), Cd.cpu().numpy())


def test_dist_device_inner_stop_matches_single_gpu():
    # eps2 > 0 on the sharded path: the stop test runs on the device, sweeps are
    # enqueued 8 at a time and launches past the stop are no-ops; the sweep counts and X match the
    # single-GPU kernel, whose inner loop is one persistent launch
    import paper_1207_1114_b200 as F
    # the c1 recipe at n = 256 with eps2 = 1e-3: the first outer iteration's inner loop stops on
    # delta after ~34 sweeps (the oracle's count), the later ones run the 300-sweep cap
    p = inputs.config1(n=256)
    p.eps2, p.max_iter2 = 1e-3, 300
    a = F.Solver(p.n, p.n_prime, p.d)
    a.set_option(F.OPT_PROJ_KERNEL, 1)                  # streaming kernel, same tiling as the shard
    a.set_graphs(p.A, p.Ap, p.B, p.Bp)
    b = _dist_solver(p)
    b.set_graphs(p.A, p.Ap, p.B, p.Bp)
    a.set_x0(p.X0)
    b.set_x0(p.X0)
    Xa, ra = a.iterate(p.alpha, p.lam, 0.0, p.eps2, 4, p.max_iter2)
    Xb, rb = b.iterate(p.alpha, p.lam, 0.0, p.eps2, 4, p.max_iter2)
    assert 8 < rb.sweeps[0] < p.max_iter2, rb.sweeps
    assert all(abs(x - y) <= 1 for x, y in zip(ra.sweeps, rb.sweeps)), (ra.sweeps, rb.sweeps)
    assert np.max(np.abs(Xa - Xb)) <= 1e-5
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)
    Xo, ro = st.iterate(p.lam, p.alpha, 0.0, p.eps2, 4, p.max_iter2)
    assert all(abs(x - y) <= 1 for x, y in zip(ro.sweeps, rb.sweeps)), (ro.sweeps, rb.sweeps)
    assert np.max(np.abs(Xb.astype(np.float64) - Xo)) <= X_TOL
    # the slack state of a sharded handle (local rows x m) round-trips through copy_y / set_y
    Y = b.copy_y()
    assert Y.shape == (p.n, max(p.n, p.n_prime))
    b.set_y(Y)
    assert np.array_equal(b.copy_y(), Y)
    a.close(); b.close()


def test_dist_nccl_timeout_aborts_and_poisons():
    # failure detection: with a 0 ms budget the first host wait finds collectives still
    # in flight, aborts the communicator and poisons the handle instead of blocking forever
    import paper_1207_1114_b200 as F
    p = inputs.config5(n=2048)
    s = _dist_solver(p)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 20)          # healthy
    s.set_option(F.OPT_NCCL_TIMEOUT_MS, 0)
    with pytest.raises(F.FastPFPError) as e:
        s.iterate(p.alpha, p.lam, 0.0, 0.0, 3, 20)
    assert e.value.status == F.ENCCL and "aborted" in str(e.value)
    with pytest.raises(F.FastPFPError) as e:
        s.iterate(p.alpha, p.lam, 0.0, 0.0, 1, 20)
    assert e.value.status == F.EPOISONED
    s.close()


@pytest.mark.parametrize("prec", [pytest.param(0, id="tf32x3"), pytest.param(3, id="int8ozaki")])
def test_dist_collective_sequence_matches_schedule(prec):
    # the collectives the library issues per outer iteration (fastpfp_dist_collectives) are exactly
    # dist.collective_schedule's — the sequence the gloo decomposition test executes on 2 ranks
    import paper_1207_1114_b200 as F
    from paper_1207_1114_b200 import dist as D
    p = inputs.config5(n=1024)
    s = _dist_solver(p)
    s.set_option(F.OPT_PRECISION, prec)
    s.set_graphs(p.A, p.Ap, p.B, p.Bp)
    s.iterate(p.alpha, p.lam, 0.0, 0.0, 2, 7)
    want = D.collective_schedule(p.n, p.n_prime, 1, prec == 3, 0.0, 7) * 2
    assert s.collectives() == want
    # eps2 > 0: sweeps are enqueued 8 at a time, each launch with its delta MAX; the log follows
    # the schedule of the enqueued launches
    s.iterate(p.alpha, p.lam, 0.0, 1e-9, 1, 20)
    log = s.collectives()
    n_sweeps = sum(1 for e in log if e == (D.ALL_REDUCE, D.NCCL_FLOAT64, D.NCCL_SUM, p.n + 1)) - 1
    assert n_sweeps in (8, 16, 20)
    assert log == D.collective_schedule(p.n, p.n_prime, 1, prec == 3, 1e-9, n_sweeps)
    s.close()
