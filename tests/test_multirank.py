"""World-size-2 CPU (gloo) coverage of the row-sharded path's host logic: the row
partition and the all-reduce of the STEP-1 projections reproduce the single-process
projection vector (the partial sums over row blocks add up to U^T a, V^T b, ...).
The projections here are formed with plain torch CPU ops as test scaffolding; on a
GPU the same partials come from svd1_project (tests/test_gpu_parity.py covers it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_08369_b200.parallel import allreduce_projection, proj_size, row_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial(U, V, a, b, g, u_lo, u_hi, v_lo, v_hi):
    m, n = U.shape[1], V.shape[1]
    out = torch.zeros(proj_size(m, n), dtype=torch.float64)
    Ul, Vl = U[u_lo:u_hi], V[v_lo:v_hi]
    out[0:m] = Ul.T @ a[u_lo:u_hi]
    for k in range(4):
        out[(1 + k) * m:(2 + k) * m] = Ul.T @ g[k, u_lo:u_hi]
    out[5 * m:5 * m + n] = Vl.T @ b[v_lo:v_hi]
    for k in range(4):
        out[5 * m + n + k] = a[u_lo:u_hi] @ g[k, u_lo:u_hi]
    out[5 * m + n + 4] = a[u_lo:u_hi] @ a[u_lo:u_hi]
    out[5 * m + n + 5] = b[v_lo:v_hi] @ b[v_lo:v_hi]
    return out


def _worker(rank, world, port, m, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    U = torch.from_numpy(rng.standard_normal((m, m)))
    V = torch.from_numpy(rng.standard_normal((n, n)))
    a, b = torch.from_numpy(rng.standard_normal(m)), torch.from_numpy(rng.standard_normal(n))
    g = torch.from_numpy(rng.standard_normal((4, m)))
    u_lo, u_hi = row_block(m, rank, world)
    v_lo, v_hi = row_block(n, rank, world)
    p = _partial(U, V, a, b, g, u_lo, u_hi, v_lo, v_hi)
    allreduce_projection(p)
    full = _partial(U, V, a, b, g, 0, m, 0, n)
    q.put((rank, float((p - full).abs().max()), float(full.abs().max()), p.numpy().tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n", [(13, 13), (8, 21)])
def test_sharded_projection_allreduce(m, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for _, err, scale, _ in res:
        assert err <= 1e-13 * scale
    # every rank holds bitwise-identical reduced projections (replicated spectral phase)
    assert res[0][3] == res[1][3]


def test_row_block_partition():
    for n in (1, 7, 4096, 16384):
        for world in (1, 2, 3, 8):
            blocks = [row_block(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in blocks]
            assert max(sizes) - min(sizes) <= 1


def _batch_worker(rank, world, port, m, n, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    U = torch.from_numpy(rng.standard_normal((m, m)))
    V = torch.from_numpy(rng.standard_normal((n, n)))
    A, B = torch.from_numpy(rng.standard_normal((K, m))), torch.from_numpy(rng.standard_normal((K, n)))
    g = torch.from_numpy(rng.standard_normal((4, m)))
    u_lo, u_hi = row_block(m, rank, world)
    v_lo, v_hi = row_block(n, rank, world)
    # the batched stream's one exchange: K projection vectors in one (K x proj) all-reduce
    projs = torch.stack([_partial(U, V, A[t], B[t], g, u_lo, u_hi, v_lo, v_hi) for t in range(K)])
    allreduce_projection(projs)
    full = torch.stack([_partial(U, V, A[t], B[t], g, 0, m, 0, n) for t in range(K)])
    q.put((rank, float((projs - full).abs().max()), float(full.abs().max()), projs.numpy().tobytes()))
    dist.destroy_process_group()


def test_sharded_batch_projection_allreduce():
    """ShardedUpdater.update_batch's exchange (world size 2, gloo): one all-reduce of
    the K stacked projection vectors gives every rank the single-process projections,
    bitwise identical across ranks."""
    world, m, n, K = 2, 11, 17, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, m, n, K, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for _, err, scale, _ in res:
        assert err <= 1e-13 * scale
    assert res[0][3] == res[1][3]


def _slice_worker(rank, world, port, n, q):
    """One rank of the sliced spectral exchange: the NCCL id from rank 0,
    then this rank's slice of per-root results gathered in place into the padded G*c
    buffer the library uses (gloo stands in for NCCL's in-place all-gather here)."""
    import oracle as O
    from paper_1707_08369_b200.parallel import shared_nccl_id, spectral_slice
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nid = shared_nccl_id(rank, world)
    rng = np.random.default_rng(3)
    d = np.sort(rng.standard_normal(n))
    z = rng.standard_normal(n)
    rho = 0.7
    k, tau = O.secular_roots_bisect(d, z, rho)          # (replicated inputs of the slice stage)
    lo, hi = spectral_slice(n, rank, world)
    c = -(-n // world)
    mine = torch.zeros(c, dtype=torch.float64)
    mine[:hi - lo] = torch.from_numpy(O.secular_w(d, z, rho, k[lo:hi], tau[lo:hi]))
    buf = torch.zeros(world * c, dtype=torch.float64)
    dist.all_gather_into_tensor(buf, mine)
    full = O.secular_w(d, z, rho, k, tau)
    q.put((rank, nid, bool(np.array_equal(buf.numpy()[:n], full)), lo, hi))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 101), (3, 100), (3, 2)])
def test_sliced_spectral_exchange(world, n):
    """World-size 2-3 (gloo): every rank receives rank 0's 128-byte NCCL id; the slices
    tile [0, n) (ragged last slice, empty slices when n < world) and their in-place gather
    reproduces the one-process per-root results bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slice_worker, args=(r, world, port, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ids = {r[1] for r in res}
    assert len(ids) == 1 and len(next(iter(ids))) == 128
    assert all(r[2] for r in res)
    assert res[0][3] == 0 and res[-1][4] == n
    assert all(res[i][4] == res[i + 1][3] for i in range(world - 1))
