"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed plumbing).

Every row of U and V is an independent right-hand side of every Cauchy apply, so rank g
owns the contiguous row blocks [g*m/G, (g+1)*m/G) of U and [g*n/G, ...) of V.  Per update
there are two kinds of exchange:

  N1  the STEP-1 projection vector (P:337 through the small-vector identities, DESIGN.md
      §4.1): each rank's partial sums (svd1_project) are all-reduced here over the torch
      process group (NCCL on GPUs);
  N2-N4  inside the library, per eigen-update: the O(n^2) spectral phase (secular roots
      P:363, Loewner weights, column norms) is sliced by index across the ranks and
      all-gathered over the plan's own NCCL communicators (svd1_config.nccl_id, created
      from the id rank 0 broadcasts here).

The tree and the expansion operators are rebuilt identically on every rank from the
gathered (bitwise-identical) spectral data; the applies touch local rows only.
"""
from __future__ import annotations


def row_block(n: int, rank: int, world: int):
    """[lo, hi) of rank's contiguous block of n rows (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def spectral_slice(n: int, rank: int, world: int):
    """[lo, hi) of the spectral indices (roots, Loewner i, norm j) rank solves: blocks of
    c = ceil(n / world), so rank r's results sit at [r c, r c + c) of the all-gather buffer
    (the library's slice_of, svd1.h)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    c = -(-n // world)
    lo = min(n, rank * c)
    return lo, min(n, lo + c)


def proj_size(m: int, n: int) -> int:
    """Length of the projection vector exchanged per update (svd1.h)."""
    return 5 * m + n + 6


def allreduce_projection(proj, group=None):
    """Sum the ranks' partial projections in place (exchange N1)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(proj, group=group)
    return proj


def shared_nccl_id(rank: int, world: int, group=None):
    """The 128-byte ncclUniqueId of the plan's communicators: made on rank 0 by libsvd1,
    broadcast to every rank over the torch process group (None on one process)."""
    if world <= 1:
        return None
    import torch.distributed as dist

    from ._lib import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class ShardedUpdater:
    """One rank's share of a row-sharded stream of rank-1 updates.

    U_loc, V_loc: this rank's row blocks (CUDA fp64, row-major); sigma, a, b full.
    Creating it is collective over the process group (the plan's NCCL communicators)."""

    def __init__(self, m, n, rank, world, eps=1e-10, stream=None, group=None, **kw):
        import torch

        from .api import Plan
        self.m, self.n, self.rank, self.world, self.group = m, n, rank, world, group
        self.u_lo, self.u_hi = row_block(m, rank, world)
        self.v_lo, self.v_hi = row_block(n, rank, world)
        self.nccl_id = shared_nccl_id(rank, world, group)
        self.plan = Plan(m, n, eps=eps, stream=stream, u_rows=self.u_hi - self.u_lo,
                         v_rows=self.v_hi - self.v_lo, u_row0=self.u_lo, v_row0=self.v_lo,
                         rank=rank, world=world, nccl_id=self.nccl_id, **kw)
        self.proj = torch.empty(proj_size(m, n), dtype=torch.float64, device="cuda")

    def update_batch(self, U_loc, sigma, V_loc, A, B):
        """A stream of K updates (A: K x m, B: K x n): every update's projections against
        the current factors, ONE all-reduce of the K projection vectors, then the
        pipelined stream on this rank's rows (svd1_update_batch_projected), whose spectral
        phases are sliced and all-gathered inside the library."""
        import torch
        from ._lib import THIN_V
        if self.world == 1:
            return self.plan.update_batch(U_loc, sigma, V_loc, A, B)
        thin = bool(self.plan.cfg.flags & THIN_V)
        K = A.shape[0]
        projs = torch.empty((K, proj_size(self.m, self.n)), dtype=torch.float64, device=A.device)
        for t in range(K):
            self.plan.project(U_loc, V_loc, A[t], B[t], projs[t])
        allreduce_projection(projs, self.group)
        return self.plan.update_batch_projected(U_loc, sigma, V_loc, projs, B if thin else None)

    def update(self, U_loc, sigma, V_loc, a, b):
        if self.world == 1:
            return self.plan.update(U_loc, sigma, V_loc, a, b)
        self.plan.project(U_loc, V_loc, a, b, self.proj)
        allreduce_projection(self.proj, self.group)
        return self.plan.update_projected(U_loc, sigma, V_loc, self.proj, a, b)
