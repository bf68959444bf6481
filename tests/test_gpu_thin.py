"""Thin right factor (SVD1_THIN_V): V kept as n x m
(plus one workspace column); the V side works in the basis [V, q], q = the direction of b
outside span(V).  Same singular triplets as the full-V update (the oracle's and the GPU's
full-V path), residual and orthogonality of the thin factors."""
import numpy as np
import pytest

import oracle as O
from compare import sigma_errors, vector_error
from synth import config_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, torch.float64)


def _thin(V, m):
    Vt = torch.zeros((V.shape[0], m + 1), dtype=torch.float64, device=DEV)
    Vt[:, :m] = T(V[:, :m])
    return Vt


@pytest.mark.parametrize("m,n,flags", [(40, 160, 0), (64, 256, P.FORCE_FMM), (300, 700, 0), (500, 2000, 0)])
def test_thin_one_update_parity(m, n, flags):
    inp = config_inputs(4, m=m, n=n, updates=1)
    U, s, V = inp["U"], inp["sigma"], inp["V"]
    a, b = inp["ab"][0]
    ref = O.svd_update(U, s, V, a, b)
    Ug, sg, Vt = T(U), T(s), _thin(V, m)
    plan = P.Plan(m, n, flags=flags | P.THIN_V)
    rep = plan.update(Ug, sg, Vt, T(a), T(b))
    assert rep["n_active"][2] <= m + 1
    se = sigma_errors(sg.cpu().numpy(), ref["sigma"])
    assert se["gram"] <= 1e-12 and se["rel_top"] <= 1e-12, se
    eu = vector_error(Ug.cpu().numpy(), ref["U"], ref["sigma"] ** 2)
    ev = vector_error(Vt[:, :m].cpu().numpy(), ref["V"][:, :m], ref["sigma"] ** 2)
    assert eu["isolated"] <= 1e-9 and ev["isolated"] <= 1e-9, (eu, ev)
    A_hat = T((U * s[None, :]) @ V[:, :m].T + np.outer(a, b))
    res = float(torch.linalg.norm(A_hat @ Vt[:, :m] - Ug * sg[None, :], dim=0).max() / sg[0])
    orth = float((Vt[:, :m].T @ Vt[:, :m] - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max())
    assert res <= 1e-10 and orth <= 1e-10, (res, orth)


@pytest.mark.parametrize("m,n,K", [(64, 256, 6), (2048, 8192, 3)])
def test_thin_stream_matches_full(m, n, K):
    """A stream of updates: thin and full V agree (U, sigma, V[:, :m]); C4 at full size."""
    inp = config_inputs(4, m=m, n=n, updates=K)
    Uf, sf, Vf = T(inp["U"]), T(inp["sigma"]), T(inp["V"])
    Ut, st, Vt = T(inp["U"]), T(inp["sigma"]), _thin(inp["V"], m)
    pf, pt = P.Plan(m, n), P.Plan(m, n, flags=P.THIN_V)
    for a, b in inp["ab"][:K]:
        pf.update(Uf, sf, Vf, T(a), T(b))
        pt.update(Ut, st, Vt, T(a), T(b))
    torch.cuda.synchronize()
    assert float((sf - st).abs().max()) <= 1e-12 * float(sf[0])
    assert float((Uf - Ut).abs().max()) <= 1e-8
    assert float((Vf[:, :m] - Vt[:, :m]).abs().max()) <= 1e-8


@pytest.mark.parametrize("m,n,K", [(64, 256, 6), (300, 1200, 5)])
def test_thin_batch_matches_sequential(m, n, K):
    """Thin V through the pipelined stream: the later b's get their coordinate along each
    update's q from the Gram matrix of the b's and the carried rows."""
    inp = config_inputs(4, m=m, n=n, updates=K)
    Ub, sb, Vb = T(inp["U"]), T(inp["sigma"]), _thin(inp["V"], m)
    Us, ss, Vs = T(inp["U"]), T(inp["sigma"]), _thin(inp["V"], m)
    pb, ps = P.Plan(m, n, flags=P.THIN_V), P.Plan(m, n, flags=P.THIN_V)
    ab = inp["ab"][:K]
    pb.update_batch(Ub, sb, Vb, T(np.stack([a for a, _ in ab])), T(np.stack([b for _, b in ab])))
    for a, b in ab:
        ps.update(Us, ss, Vs, T(a), T(b))
    torch.cuda.synchronize()
    assert float((sb - ss).abs().max()) <= 1e-12 * float(ss[0])
    assert float((Ub - Us).abs().max()) <= 1e-8
    assert float((Vb[:, :m] - Vs[:, :m]).abs().max()) <= 1e-8


def test_thin_b_in_span():
    """b inside span(V[:, :m]): no null-space component (beta_perp = 0), the extra
    coordinate has zero weight and deflates; same result as the full-V path."""
    m, n = 48, 160
    inp = config_inputs(4, m=m, n=n, updates=1)
    U, s, V = inp["U"], inp["sigma"], inp["V"]
    a, _ = inp["ab"][0]
    b = V[:, :m] @ np.random.default_rng(5).standard_normal(m)
    Uf, sf, Vf = T(U), T(s), T(V)
    P.Plan(m, n).update(Uf, sf, Vf, T(a), T(b))
    Ut, st, Vt = T(U), T(s), _thin(V, m)
    rep = P.Plan(m, n, flags=P.THIN_V).update(Ut, st, Vt, T(a), T(b))
    torch.cuda.synchronize()
    assert rep["n_deflated"][2] >= 1
    assert bool(torch.isfinite(Vt).all())
    assert float((sf - st).abs().max()) <= 1e-12 * float(sf[0])
    assert float((Uf - Ut).abs().max()) <= 1e-8 and float((Vf[:, :m] - Vt[:, :m]).abs().max()) <= 1e-8


@pytest.mark.parametrize("name", ["tiny13", "tiny25", "b_null_space"])
def test_thin_edge_cases(name):
    """Thin right factor on the rectangular edge recipes (synth/edge.py): m = 1 and 2, and b
    entirely in the null space of A's rows (V^T b = 0 on the first m columns: the whole V-side
    update lives in the extra direction q)."""
    from synth import edge_case
    U, s, V, a, b = edge_case(name)
    m, n = U.shape[0], V.shape[0]
    ref = O.svd_update(U, s, V, a, b)
    Ug, sg, Vt = T(U), T(s), _thin(V, m)
    plan = P.Plan(m, n, flags=P.THIN_V)
    plan.update(Ug, sg, Vt, T(a), T(b))
    se = sigma_errors(sg.cpu().numpy(), ref["sigma"])
    assert se["gram"] <= 1e-12 and se["rel_top"] <= 1e-12, se
    eu = vector_error(Ug.cpu().numpy(), ref["U"], ref["sigma"] ** 2)
    ev = vector_error(Vt[:, :m].cpu().numpy(), ref["V"][:, :m], ref["sigma"] ** 2)
    assert max(eu["isolated"], eu["cluster"], ev["isolated"], ev["cluster"]) <= 1e-9, (eu, ev)
    A_hat = T((U * s[None, :]) @ V[:, :m].T + np.outer(a, b))
    res = float(torch.linalg.norm(A_hat @ Vt[:, :m] - Ug * sg[None, :], dim=0).max() / sg[0])
    orth = float((Vt[:, :m].T @ Vt[:, :m] - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max())
    assert res <= 1e-10 and orth <= 1e-10, (res, orth)
