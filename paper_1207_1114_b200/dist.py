"""Host-side plumbing of the row-sharded FastPFP path (one process per GPU).

The arithmetic and the collectives of the sharded outer iteration run inside the C-ABI library
(fastpfp_create_dist: NCCL all-gather of U, all-reduces of column sums / mu / rho over NVLink). This
module only does what belongs to the host: the row partition, the NCCL-id bootstrap over the torch
process group, and slicing the local inputs. No method arithmetic lives here.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RowShard:
    rank: int
    world: int
    n: int            # global rows (nodes of G)
    row0: int         # first global row owned by this rank
    rows: int         # rows owned (n / world)

    @property
    def sl(self) -> slice:
        return slice(self.row0, self.row0 + self.rows)


def row_partition(n: int, n_prime: int, world: int, rank: int) -> RowShard:
    """Block row partition used by fastpfp_create_dist: equal blocks of n/world rows, each a
    multiple of 32 (the GEMM2 K-block), and n >= n' (slack columns stay local, reading A1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if n < n_prime:
        raise ValueError("row sharding needs n >= n' (swap the graphs: transpose equivariance, reading A1)")
    if n % world or (n // world) % 32:
        raise ValueError(f"n={n} must split into {world} blocks that are multiples of 32")
    rows = n // world
    return RowShard(rank, world, n, rank * rows, rows)


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def broadcast_uid(uid: bytes | None, rank: int, world: int, group=None) -> bytes:
    """Broadcast the 128-byte NCCL id from rank 0 over the torch process group (any backend)."""
    if world == 1:
        assert uid is not None
        return uid
    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf[:] = torch.frombuffer(bytearray(uid), dtype=torch.uint8)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        b = buf.to(dev)
        dist.broadcast(b, src=0, group=group)
        buf = b.cpu()
    else:
        dist.broadcast(buf, src=0, group=group)
    return bytes(buf.numpy().tobytes())


def make_solver(n: int, n_prime: int, d: int, rank: int | None = None, world: int | None = None,
                group=None):
    """Create this rank's sharded Solver (collective over the torch process group)."""
    import paper_1207_1114_b200 as F
    r, w = env_rank_world()
    rank = r if rank is None else rank
    world = w if world is None else world
    row_partition(n, n_prime, world, rank)      # validate before any collective
    uid = F.nccl_unique_id() if rank == 0 else None
    uid = broadcast_uid(uid, rank, world, group)
    return F.Solver(n, n_prime, d, dist=(rank, world, uid))


def local_inputs(problem, shard: RowShard):
    """(A rows, A', B rows, B') of this rank as contiguous float32 arrays."""
    A = np.ascontiguousarray(problem.A[shard.sl])
    B = None if problem.B is None else np.ascontiguousarray(problem.B[shard.sl])
    return A, problem.Ap, B, problem.Bp


# ------------------------------------------------------------------------------------------------
# The collective schedule of one sharded outer iteration
# ------------------------------------------------------------------------------------------------
# Entries are (kind, dtype, op, count) with NCCL's enum values, the encoding
# fastpfp_dist_collectives reports: kind 0 = all-reduce, 1 = all-gather; op -1 for all-gathers.
ALL_REDUCE, ALL_GATHER = 0, 1
NCCL_INT8, NCCL_UINT32, NCCL_FLOAT32, NCCL_FLOAT64 = 0, 3, 7, 8
NCCL_SUM, NCCL_MAX = 0, 2


def _round_up(x: int, q: int) -> int:
    return (x + q - 1) // q * q


def collective_schedule(n: int, n_prime: int, world: int, int8: bool, eps2: float, sweeps: int):
    """The collectives one outer iteration of the row-sharded path issues, in order, when its inner
    loop makes `sweeps` sweep launches (the fixed count when eps2 == 0):
      GEMM1 -> [int8: MAX of U's per-row |max| (n' uint32); all-gather of U's 3 digit planes
               (n' x round_up(n/P, 128) int8 each) | TF32: all-gather of U's big and small parts
               (n' x round_up(n/P, 32) fp32 each)] -> GEMM2 ->
      sums pass: SUM of [column sums | sigma] (m + 1 fp64) ->
      per sweep: SUM of [column sums | sigma]; MAX of delta (1 fp64) when eps2 > 0 or on the last
      sweep -> MAX of mu (1 fp64) -> MAX of rho (1 fp64)."""
    rows = n // world
    m = max(n, n_prime)
    out = []
    if int8:
        out.append((ALL_REDUCE, NCCL_UINT32, NCCL_MAX, n_prime))
        out += [(ALL_GATHER, NCCL_INT8, -1, n_prime * _round_up(rows, 128))] * 3
    else:
        out += [(ALL_GATHER, NCCL_FLOAT32, -1, n_prime * _round_up(rows, 32))] * 2
    out.append((ALL_REDUCE, NCCL_FLOAT64, NCCL_SUM, m + 1))
    for s in range(sweeps):
        out.append((ALL_REDUCE, NCCL_FLOAT64, NCCL_SUM, m + 1))
        if eps2 > 0.0 or s + 1 == sweeps:
            out.append((ALL_REDUCE, NCCL_FLOAT64, NCCL_MAX, 1))
    out.append((ALL_REDUCE, NCCL_FLOAT64, NCCL_MAX, 1))
    out.append((ALL_REDUCE, NCCL_FLOAT64, NCCL_MAX, 1))
    return out
