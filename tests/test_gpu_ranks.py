"""Multi-rank spectral phase on the one GPU available: the
sliced kernels, the padded all-gather layout and the host logic, through the C ABI.

  * SVD1_EMULATE_RANKS: one process computes every rank's slice of the roots (P:363
    STEP 2), Loewner weights and column norms -- the all-gather becomes a concatenation
    in place -- and the result must be BITWISE that of world = 1 (each index is computed
    by the same code whatever slice it falls in);
  * SVD1_FORCE_NCCL with world = 1: the plan's NCCL communicators and in-place
    all-gathers run for real (libnccl.so.2 opened by the library), bitwise as without.
Ranks on separate GPUs cannot be run here (one GPU per call); the exchange itself is
covered on CPU by tests/test_multirank.py (gloo)."""
import numpy as np
import pytest

from synth import config_inputs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, torch.float64)


def _run(inp, K, batch, **plan_kw):
    U, s, V = T(inp["U"]), T(inp["sigma"]), T(inp["V"])
    plan = P.Plan(U.shape[0], V.shape[0], **plan_kw)
    ab = inp["ab"][:K]
    if batch:
        reps = plan.update_batch(U, s, V, T(np.stack([a for a, _ in ab])), T(np.stack([b for _, b in ab])))
    else:
        reps = [plan.update(U, s, V, T(a), T(b)) for a, b in ab]
    torch.cuda.synchronize()
    plan.close()
    return U, s, V, reps


def _bitwise(x, y):
    return all(torch.equal(a, b) for a, b in zip(x[:3], y[:3]))


@pytest.mark.parametrize("cfg,m,n,K,flags", [
    (3, 256, 256, 3, P.FORCE_FMM),                  # graded: FMM applies, direct secular
    (5, 203, 203, 2, P.FORCE_FMM),                  # duplicated sigma (deflation), ragged slices
    (4, 40, 131, 2, 0),                             # rectangular: V's null space, n_a != N
    (3, 515, 515, 2, P.FORCE_FMM | P.SECULAR_FMM),  # the FMM secular solve, sliced
])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_ranks_bitwise_per_update(cfg, m, n, K, flags, world):
    inp = config_inputs(cfg, m=m, n=n, updates=K)
    ref = _run(inp, K, False, flags=flags)
    got = _run(inp, K, False, flags=flags | P.EMULATE_RANKS, world=world)
    assert _bitwise(ref, got)
    assert [r["n_active"] for r in ref[3]] == [r["n_active"] for r in got[3]]


@pytest.mark.parametrize("world", [2, 5])
def test_emulated_ranks_bitwise_batch(world):
    """The pipelined stream (svd1_update_batch, what bench.py times) with sliced spectral
    phases: bitwise the world = 1 stream."""
    inp = config_inputs(3, m=384, n=384, updates=5)
    ref = _run(inp, 5, True, flags=P.FORCE_FMM | P.SECULAR_FMM)
    got = _run(inp, 5, True, flags=P.FORCE_FMM | P.SECULAR_FMM | P.EMULATE_RANKS, world=world)
    assert _bitwise(ref, got)


def test_nccl_communicator_path_world1():
    """The NCCL path for real on one GPU: communicator creation from a unique id (rank 0),
    the split for the second side chain, grouped in-place all-gathers of every stage."""
    inp = config_inputs(3, m=320, n=320, updates=3)
    ref = _run(inp, 3, True, flags=P.FORCE_FMM)
    nid = P.nccl_unique_id()
    got = _run(inp, 3, True, flags=P.FORCE_FMM | P.FORCE_NCCL, rank=0, world=1, nccl_id=nid)
    assert _bitwise(ref, got)
    got1 = _run(inp, 2, False, flags=P.FORCE_FMM | P.FORCE_NCCL, rank=0, world=1, nccl_id=P.nccl_unique_id())
    ref1 = _run(inp, 2, False, flags=P.FORCE_FMM)
    assert _bitwise(ref1, got1)


def test_rank_config_errors():
    with pytest.raises(P.SVD1Error) as e:  # world > 1 needs a communicator id (or emulation)
        P.Plan(64, 64, world=2, rank=0)
    assert e.value.code == 1
    with pytest.raises(P.SVD1Error) as e:
        P.Plan(64, 64, world=2, rank=2, flags=P.EMULATE_RANKS)
    assert e.value.code == 1


@pytest.mark.parametrize("name", ["all_equal", "unbalanced", "scaled_down"])
def test_emulated_ranks_bitwise_edge(name):
    """Sliced spectral phases on the edge recipes whose host decisions are new (the D9
    balance, the D5 pairing of a 46-column cluster): bitwise the world = 1 result."""
    from synth import edge_case
    U, s, V, a, b = edge_case(name, m=96)
    inp = dict(U=U, sigma=s, V=V, ab=[(a, b)])
    ref = _run(inp, 1, False, flags=P.FORCE_FMM)
    got = _run(inp, 1, False, flags=P.FORCE_FMM | P.EMULATE_RANKS, world=3)
    assert _bitwise(ref, got)
