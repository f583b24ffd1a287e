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
