"""Fused per-side pass (SVD1_FUSED_SIDE): each side's two
applies run row chunk by row chunk.  Rows are independent right-hand sides and every chunk
runs the same kernels on the same operators, so the factors must be BITWISE those of the
unfused path (whose parity with the oracle tests/test_gpu_parity.py and
tests/test_gpu_fullsize.py establish).  Small cases use 128-row chunks (several chunks,
ragged last chunk; set before the library first reads it).  bench.py --fused runs the
default L2-sized chunks."""
import os

import numpy as np
import pytest

os.environ.setdefault("SVD1_FUSED_ROWS", "128")  # several chunks even in the small cases
from synth import config_inputs  # noqa: E402

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, torch.float64) if isinstance(x, np.ndarray) else x.clone()


def _run(inp, K, batch, flags, thin=False):
    U, s = T(inp["U"]), T(inp["sigma"])
    m, n = U.shape[0], inp["V"].shape[0]
    if thin:
        V = torch.zeros((n, m + 1), dtype=torch.float64, device=DEV)
        V[:, :m] = T(inp["V"])[:, :m]
    else:
        V = T(inp["V"])
    plan = P.Plan(m, n, flags=flags)
    ab = inp["ab"][:K]
    if batch:
        A = torch.stack([T(a) if isinstance(a, np.ndarray) else a for a, _ in ab]).to(DEV)
        B = torch.stack([T(b) if isinstance(b, np.ndarray) else b for _, b in ab]).to(DEV)
        reps = plan.update_batch(U, s, V, A, B)
    else:
        reps = [plan.update(U, s, V, T(a), T(b)) for a, b in ab]
    torch.cuda.synchronize()
    plan.close()
    return U, s, V, reps


@pytest.mark.parametrize("cfg,m,n,K,flags,batch,thin", [
    (3, 700, 700, 3, P.FORCE_FMM, False, False),   # graded, several 128-row chunks, ragged tail
    (3, 700, 700, 4, P.FORCE_FMM, True, False),    # the pipelined stream
    (5, 300, 300, 2, P.FORCE_FMM, True, False),    # duplicates: Householder groups, pairing rotations
    (4, 200, 520, 3, 0, True, False),              # rectangular full V: null-space Householder
    (4, 200, 520, 3, P.THIN_V, True, True),        # thin V
    (2, 257, 257, 2, P.FORCE_DIRECT, False, False),  # direct apply in chunks
])
def test_fused_side_bitwise(cfg, m, n, K, flags, batch, thin):
    inp = config_inputs(cfg, m=m, n=n, updates=K)
    ref = _run(inp, K, batch, flags, thin)
    got = _run(inp, K, batch, flags | P.FUSED_SIDE, thin)
    for a, b in zip(ref[:3], got[:3]):
        assert torch.equal(a, b), float((a - b).abs().max())


def test_fused_side_c3_full_size():
    """The full-size C3 stream (default, L2-sized chunks) through svd1_update_batch."""
    inp = config_inputs(3, device=DEV, updates=6)
    ref = _run(inp, 6, True, 0)
    got = _run(inp, 6, True, P.FUSED_SIDE)
    for a, b in zip(ref[:3], got[:3]):
        assert torch.equal(a, b), float((a - b).abs().max())
    assert all(r["allocations"] == 0 for r in got[3])
