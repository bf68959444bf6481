"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(one process, plan on the current stream, FMM on): sampled output rows against the
oracle's O8 large-n mode (exact spectral phase, products on the sampled rows; rows
are independent), plus invariants at full size computed on the GPU (fp64 GEMMs,
verification only).  Q30: for a second update the oracle is fed the GPU's factors."""
import numpy as np
import pytest

import oracle as O
from compare import assert_parity, log_parity, sigma_errors, vector_error_rows
from synth import config_inputs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def _invariants(A_hat, Ug, sg, Vg):
    m = Ug.shape[0]
    res = float(torch.linalg.norm(A_hat @ Vg[:, :m] - Ug * sg[None, :], dim=0).max() / sg[0])
    Im = torch.eye(m, dtype=torch.float64, device=DEV)
    In = torch.eye(Vg.shape[0], dtype=torch.float64, device=DEV)
    orth = max(float((Ug.T @ Ug - Im).abs().max()), float((Vg.T @ Vg - In).abs().max()))
    return res, orth


def _sampled_parity(cfg, updates, n_rows=96):
    inp = config_inputs(cfg, device=DEV, updates=updates)
    m, n = inp["cfg"]["m"], inp["cfg"]["n"]
    Ug, sg, Vg = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
    A = (Ug * sg[None, :]) @ Vg[:, :m].T
    plan = P.Plan(m, n, eps=inp["cfg"]["eps"])
    rng = np.random.default_rng(99)
    ru = np.sort(rng.choice(m, size=min(n_rows, m), replace=False))
    rv = np.sort(rng.choice(n, size=min(n_rows, n), replace=False))
    out = []
    for (a, b) in inp["ab"]:
        U0, s0, V0 = Ug.cpu().numpy(), sg.cpu().numpy(), Vg.cpu().numpy()
        ref = O.svd_update(U0, s0, V0, a, b, sign_rule="probe", rows=(ru, rv))
        rep = plan.update(Ug, sg, Vg, torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV))
        A = A + torch.outer(torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV))
        se = sigma_errors(sg.cpu().numpy(), ref["sigma"])
        eu = vector_error_rows(Ug.cpu().numpy()[ru], ref["U"], ref["sigma"] ** 2)
        ev = vector_error_rows(Vg.cpu().numpy()[rv], ref["V"], ref["info"]["Dv_hat"])
        res, orth = _invariants(A, Ug, sg, Vg)
        out.append(dict(sigma=se, U=eu, V=ev, res=res, orth=orth, rep=rep))
    return out


def test_c3_full_size_two_updates():
    for t, r in enumerate(_sampled_parity(3, 2)):
        assert r["rep"]["fmm_used"] == [1, 1, 1, 1]
        assert_parity(f"C3 full size, svd1_update, step {t}", r)


def test_c4_full_size_one_update():
    """m = 2048, n = 8192: rectangular, the 6144-dim null space of D_v deflated by
    Householder on the V side (H10)."""
    (r,) = _sampled_parity(4, 1, n_rows=64)
    assert r["rep"]["n_deflated"][2] >= 6143
    assert_parity("C4 full size, svd1_update, step 0", r)


def _batch_prefix(inp, plan, t):
    """Factors after updates 0..t-1 of the stream through ONE svd1_update_batch call (the
    API bench.py times: carried projection rows, few-rows Cauchy products, FMM applies,
    the FMM secular solve at these sizes)."""
    U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
    if t > 0:
        A = torch.stack([torch.from_numpy(a) for a, _ in inp["ab"][:t]]).to(DEV)
        B = torch.stack([torch.from_numpy(b) for _, b in inp["ab"][:t]]).to(DEV)
        reps = plan.update_batch(U, s, V, A, B)
    else:
        reps = []
    torch.cuda.synchronize()
    return U, s, V, reps


def _batch_step_parity(cfg, steps, n_rows=96):
    """Q30 one-step parity of the timed path: for update t of the stream, the oracle (O8:
    exact spectral phase, explicit products on sampled rows) is fed the factors of the
    GPU's batch run over updates 0..t-1, and compared with the GPU's batch run over
    updates 0..t, in which update t is the LAST of the call (its projections came through
    every earlier update's transforms as carried rows)."""
    inp = config_inputs(cfg, device=DEV)
    m, n = inp["cfg"]["m"], inp["cfg"]["n"]
    plan = P.Plan(m, n, eps=inp["cfg"]["eps"])
    rng = np.random.default_rng(99)
    ru = np.sort(rng.choice(m, size=min(n_rows, m), replace=False))
    rv = np.sort(rng.choice(n, size=min(n_rows, n), replace=False))
    out = []
    for t in steps:
        Up, sp, Vp, _ = _batch_prefix(inp, plan, t)
        Un, sn, Vn, reps = _batch_prefix(inp, plan, t + 1)
        a, b = inp["ab"][t]
        ref = O.svd_update(Up.cpu().numpy(), sp.cpu().numpy(), Vp.cpu().numpy(), a, b, sign_rule="probe",
                           rows=(ru, rv))
        del Up, Vp
        A = (inp["U"] * inp["sigma"][None, :]) @ inp["V"][:, :m].T
        for q in range(t + 1):
            A = A + torch.outer(torch.from_numpy(inp["ab"][q][0]).to(DEV), torch.from_numpy(inp["ab"][q][1]).to(DEV))
        res, orth = _invariants(A, Un, sn, Vn)
        del A
        r = dict(sigma=sigma_errors(sn.cpu().numpy(), ref["sigma"]),
                 U=vector_error_rows(Un.cpu().numpy()[ru], ref["U"], ref["sigma"] ** 2),
                 V=vector_error_rows(Vn.cpu().numpy()[rv], ref["V"], ref["info"]["Dv_hat"]),
                 res=res, orth=orth, rep=reps[-1], t=t)
        out.append(r)
    plan.close()
    return out


def test_c3_batch_stream_oracle_parity():
    """C3 at full size (m = n = 4096, graded spectrum, 16-update stream) through
    svd1_update_batch -- the configuration bench.py times -- against the oracle, one step
    at a time (Q30) at the stream's first carried-row update, its middle and its end."""
    for r in _batch_step_parity(3, (1, 8, 15)):
        assert r["rep"]["fmm_used"] == [1, 1, 1, 1]
        assert r["rep"]["allocations"] == 0
        assert_parity(f"C3 full size, svd1_update_batch, step {r['t']}", r, fmm_levels=r["rep"]["fmm_levels"],
                      n_active=r["rep"]["n_active"])


def test_c5_batch_oracle_parity():
    """C5 at full size (m = n = 16384, sigma ~ U[1,100] with 5% bitwise duplicates)
    through svd1_update_batch, update 1 of the stream (carried rows) against the oracle's
    O8 mode on 96 sampled rows: exact spectral phase (bisection over all 16384 roots of
    each of the four eigen-updates), duplicated sigma deflated by Householder, clusters
    compared through their projectors (Q27)."""
    (r,) = _batch_step_parity(5, (1,))
    assert sum(r["rep"]["n_deflated"]) > 0
    assert_parity("C5 full size, svd1_update_batch, step 1", r, n_deflated=r["rep"]["n_deflated"],
                  pair_rotations=r["rep"]["pair_rotations"])


def test_c5_full_size_invariants():
    """m = n = 16384, sigma ~ U[1,100] with 5% bitwise duplicates: invariants at full
    size (the oracle's O(n^2 * 64) bisection at this n is too slow for the suite):
    residual, orthogonality, Weyl interlacing and the Frobenius identity."""
    inp = config_inputs(5, device=DEV, updates=1)
    m = n = 16384
    Ug, sg, Vg = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
    s_old = sg.clone()
    a, b = (torch.from_numpy(x).to(DEV) for x in inp["ab"][0])
    xa, yb = Ug.T @ a, Vg.T @ b
    A = (Ug * sg[None, :]) @ Vg.T + torch.outer(a, b)
    plan = P.Plan(m, n, eps=1e-10)
    rep = plan.update(Ug, sg, Vg, a, b)
    assert sum(rep["n_deflated"][:1]) > 0  # duplicated sigma -> Householder deflation
    res, orth = _invariants(A, Ug, sg, Vg)
    assert res <= 1e-10 and orth <= 1e-10, (res, orth)
    sh, so = sg.cpu().numpy(), s_old.cpu().numpy()
    tol = 1e-12 * sh[0]
    assert np.all(sh[1:] <= so[:-1] + tol) and np.all(so[1:] <= sh[:-1] + tol)
    frob = float((s_old ** 2).sum() + 2 * (xa * s_old * yb).sum() + (a @ a) * (b @ b))
    assert float((sg ** 2).sum()) == pytest.approx(frob, rel=1e-12)
