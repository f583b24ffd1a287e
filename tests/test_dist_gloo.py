"""World-size-2 CPU (gloo) tests of the row-sharded path's host logic and decomposition.

The decomposition below issues its collectives through `Schedule`, which asserts that they are, in
kind, reduction and element count, exactly `dist.collective_schedule` — the sequence the library's
sharded iteration is checked to issue on the GPU (fastpfp_dist_collectives).

The sharded GPU iteration (fastpfp_create_dist) exchanges exactly three things per outer iteration:
an all-gather of U_r = A' X_r^T, an all-reduce SUM of the column sums (+ sigma) per sweep, and
all-reduces MAX of mu and rho. Here two gloo ranks run that same decomposition in
fp64 numpy with real torch.distributed collectives, using the product's partition / NCCL-id
bootstrap helpers (paper_1207_1114_b200.dist), and must reproduce the unsharded oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import fastpfp as O
from paper_1207_1114_b200 import dist as D
from paper_1207_1114_b200 import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather_cols(U_r, world):
    parts = [torch.zeros_like(torch.from_numpy(U_r)) for _ in range(world)]
    tdist.all_gather(parts, torch.from_numpy(U_r))
    return np.concatenate([p.numpy() for p in parts], axis=1)


def _allreduce(x, op):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    tdist.all_reduce(t, op=op)
    return t.numpy()


class Schedule:
    """Checks each collective the decomposition makes against D.collective_schedule, the sequence
    the library issues (tests/test_gpu_dist.py::test_dist_collective_sequence_matches_schedule)."""

    def __init__(self):
        self.log = []

    def allreduce(self, x, op, count):
        self.log.append((D.ALL_REDUCE, D.NCCL_MAX if op == tdist.ReduceOp.MAX else D.NCCL_SUM, count))
        return _allreduce(x, op)

    def allgather(self, U_r, world, count, parts):
        self.log += [(D.ALL_GATHER, -1, count)] * parts
        return _allgather_cols(U_r, world)


def sharded_outer(sh, A_r, Ap, K_r, X_r, Y_r, lam, alpha, eps2, max_iter2, m, sched):
    """One outer iteration of Algorithm 1 in the sharded decomposition (int8 path's
    collectives: row-scale MAX, digit-plane all-gather, per-sweep column sums, MAX of delta, mu, rho)."""
    npr = Ap.shape[0]
    U_r = Ap @ X_r.T                                   # GEMM1, local
    # int8 path: U's per-row scale must be global (one exponent per row of the gathered U): the
    # all-reduce MAX of the local row maxima equals the row maxima of the full U
    rowmax = sched.allreduce(np.max(np.abs(U_r), axis=1), tdist.ReduceOp.MAX, npr)
    U = sched.allgather(U_r, sh.world, npr * D._round_up(sh.rows, 128), 3)   # U's 3 digit planes
    assert np.array_equal(rowmax, np.max(np.abs(U), axis=1))
    Y_r[:, :npr] = A_r @ U.T + lam * K_r               # GEMM2 (+ lambda K), local rows
    cs = sched.allreduce(np.append(Y_r.sum(0), Y_r.sum()), tdist.ReduceOp.SUM, m + 1)
    c, sigma = cs[:m], cs[m]
    r = Y_r.sum(1)
    sweeps = 0
    while True:
        Z = np.maximum(Y_r + ((1.0 + sigma / m) / m - r / m)[:, None] - (c / m)[None, :], 0.0)
        delta_loc = np.max(np.abs(Z - Y_r))
        Y_r[:] = Z
        cs = sched.allreduce(np.append(Y_r.sum(0), Y_r.sum()), tdist.ReduceOp.SUM, m + 1)
        delta = sched.allreduce(np.array([delta_loc]), tdist.ReduceOp.MAX, 1)[0]
        c, sigma = cs[:m], cs[m]
        r = Y_r.sum(1)
        sweeps += 1
        if delta < eps2 or sweeps >= max_iter2:
            break
    Xt = (1 - alpha) * X_r + alpha * Y_r[:, :npr]
    mu = sched.allreduce(np.array([Xt.max()]), tdist.ReduceOp.MAX, 1)[0]
    Xn = Xt / mu
    rho = sched.allreduce(np.array([np.max(np.abs(Xn - X_r))]), tdist.ReduceOp.MAX, 1)[0]
    # the same collectives, in the same order, as the library's sharded iteration
    want = [(k, op, cnt) for (k, _, op, cnt) in D.collective_schedule(sh.n, npr, sh.world, True, eps2, sweeps)]
    assert sched.log == want, (sched.log[:6], want[:6])
    sched.log.clear()
    return Xn, rho, sweeps


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # NCCL-id bootstrap helper (any backend): rank 0's bytes reach every rank
        uid = bytes(range(128)) if rank == 0 else None
        got = D.broadcast_uid(uid, rank, world)
        assert got == bytes(range(128))
        for (n, npr, d) in [(64, 64, 3), (64, 50, 2)]:
            p = inputs.planted_unequal(11 + npr, n, npr, d=d) if n != npr else \
                inputs.config5(n=n, d=d)
            sh = D.row_partition(n, npr, world, rank)
            A_r, Ap, B_r, Bp = D.local_inputs(p, sh)
            K_r = O.affinity(B_r, Bp, sh.rows, npr)
            m = max(n, npr)
            X_r = np.full((sh.rows, npr), 1.0 / (n * npr))
            Y_r = np.zeros((sh.rows, m))
            st = O.FastPFP(p.A, p.Ap, p.B, p.Bp)
            for t in range(6):
                X_r, rho, sw = sharded_outer(sh, np.asarray(A_r, np.float64), np.asarray(Ap, np.float64),
                                             K_r, X_r, Y_r, p.lam, p.alpha, 1e-7, 40, m, Schedule())
                Xo, rep = st.iterate(p.lam, p.alpha, 0.0, 1e-7, 1, 40)
                assert np.max(np.abs(X_r - Xo[sh.sl])) < 1e-10, (n, npr, t)
                assert abs(rho - rep.rho[0]) < 1e-10 and sw == rep.sweeps[0]
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        tdist.destroy_process_group()


def test_row_partition_rules():
    sh = D.row_partition(16384, 16384, 8, 3)
    assert (sh.row0, sh.rows) == (6144, 2048)
    with pytest.raises(ValueError):
        D.row_partition(1000, 1000, 8, 0)      # 125 rows per rank is not a multiple of 32
    with pytest.raises(ValueError):
        D.row_partition(800, 1000, 2, 0)       # n < n'
    with pytest.raises(ValueError):
        D.row_partition(64, 64, 2, 2)


def test_sharded_decomposition_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
