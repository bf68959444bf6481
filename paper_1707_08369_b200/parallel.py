"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed plumbing).

Every row of U and V is an independent right-hand side of every Cauchy apply, so
rank g owns the contiguous row blocks [g*m/G, (g+1)*m/G) of U and [g*n/G, ...) of V.
The only exchange of the update is the STEP-1 projection vector (P:337 through the
small-vector identities): each rank computes its partial sums with
svd1_project, an all-reduce (NCCL on GPUs) sums them, and svd1_update_projected then
replicates the O(n^2) spectral phase (deterministic, identical on every rank) and
applies the plan to its own rows.  DESIGN.md §7.
"""
from __future__ import annotations


def row_block(n: int, rank: int, world: int):
    """[lo, hi) of rank's contiguous block of n rows (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def proj_size(m: int, n: int) -> int:
    """Length of the projection vector exchanged per update (svd1.h)."""
    return 5 * m + n + 6


def allreduce_projection(proj, group=None):
    """Sum the ranks' partial projections in place (the path's one collective)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(proj, group=group)
    return proj


class ShardedUpdater:
    """One rank's share of a row-sharded stream of rank-1 updates.

    U_loc, V_loc: this rank's row blocks (CUDA fp64, row-major); sigma, a, b full."""

    def __init__(self, m, n, rank, world, eps=1e-10, stream=None, group=None, **kw):
        import torch

        from .api import Plan
        self.m, self.n, self.rank, self.world, self.group = m, n, rank, world, group
        self.u_lo, self.u_hi = row_block(m, rank, world)
        self.v_lo, self.v_hi = row_block(n, rank, world)
        self.plan = Plan(m, n, eps=eps, stream=stream, u_rows=self.u_hi - self.u_lo,
                         v_rows=self.v_hi - self.v_lo, u_row0=self.u_lo, v_row0=self.v_lo, **kw)
        self.proj = torch.empty(proj_size(m, n), dtype=torch.float64, device="cuda")

    def update_batch(self, U_loc, sigma, V_loc, A, B):
        """A stream of K updates (A: K x m, B: K x n): every update's projections against
        the current factors, ONE all-reduce of the K projection vectors, then the
        pipelined stream on this rank's rows (svd1_update_batch_projected)."""
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
