"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Tolerances: north star + readings Q23, Q26-Q29."""
import numpy as np
import pytest

import oracle as O
from compare import assert_parity, sigma_errors, vector_error
from synth import config_inputs, interlaced_cauchy, random_secular

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def T(x, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, dt)


def N(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def plan():
    return P.Plan(8, 8, eps=1e-10)


# ------------------------------------------------------------------ K2
CASES = [(n, kind, s) for n in (1, 2, 5, 33, 257, 1000) for kind in ("gaussian", "graded", "uniform")
         for s in (1.0, -1.0)]


@pytest.mark.parametrize("n,kind,sgn", CASES)
def test_secular_parity(plan, n, kind, sgn):
    rng = np.random.default_rng(n * 7 + len(kind))
    d, z, rho = random_secular(n, rng, kind=kind)
    rho = sgn * abs(rho)
    dfl = O.deflate(d, z, rho)
    d, z = dfl.d[dfl.active], dfl.z[dfl.active]
    n = d.size
    ko, to = O.secular_roots_bisect(d, z, rho)
    kg, tg, iters = plan.secular_solve(T(d), T(z), rho)
    kg, tg = N(kg).astype(np.int64), N(tg)
    # same root in gap form: mu_g - mu_o = (d[kg] - d[ko]) + tg - to
    diff = ((d[kg] - d[ko]) + tg) - to
    scale = np.minimum(np.abs(to), np.abs(tg))
    assert np.max(np.abs(diff) / scale) <= 2e-12, (np.max(np.abs(diff) / scale), iters)
    # the GPU roots are inside the rounding band of w (oracle's evaluation)
    w = O.secular_w(d, z, rho, kg, tg)
    terms = np.abs(z[None, :] ** 2 / ((d[None, :] - d[kg][:, None]) - tg[:, None]))
    assert np.all(np.abs(w) <= 64 * n * O.EPS * (1 + abs(rho) * terms.sum(axis=1)))
    assert iters <= 40


@pytest.mark.parametrize("n,kind", [(3, "gaussian"), (300, "graded"), (1000, "uniform"), (2500, "uniform"),
                                    (1500, "wide"), (8192, "wide")])
def test_loewner_and_colnorm_parity(plan, n, kind):
    """(2500: full shared-memory tiles with and without the diagonal; 'wide': products of a
    few gaps overflow between the fast renormalisations -> the per-index / per-chunk frexp
    redo, in the warp kernel (n < 8192) and the chunked kernel (8192))"""
    rng = np.random.default_rng(11 + n)
    d, z, rho = random_secular(n, rng, kind=kind)
    k, tau = O.secular_roots_bisect(d, z, rho)
    zo = O.loewner_zhat(d, k, tau, rho, z)
    zg = N(plan.loewner(T(d), T(k, torch.int32), T(tau), rho, T(z)))
    assert np.max(np.abs(zg / zo - 1)) <= 1e-12
    if n > 4096:
        return  # (the norms' explicit X would be n^2 doubles; covered at the other sizes)
    _, cn = O.cauchy_X(d, k, tau, zo)
    cg = N(plan.colnorms(T(d), T(k, torch.int32), T(tau), T(zo)))
    assert np.max(np.abs(cg / cn - 1)) <= 1e-13


# ------------------------------------------------------------------ K11 / FMM
def _abs_scale(u_in, d, k, tau, zh, cs):
    """E_rj = cs_j sum_i |U_ri zhat_i| / |(d_i - d_kj) - tau_j| (error scale of the sum)."""
    inv = 1.0 / np.abs((d[:, None] - d[k][None, :]) - tau[None, :])
    return (np.abs(u_in * zh[None, :]) @ inv) * np.abs(cs)[None, :]


@pytest.mark.parametrize("rows,n,sgn", [(1, 1, 1.0), (7, 5, 1.0), (300, 200, -1.0), (129, 1000, 1.0)])
def test_cauchy_apply_direct(rows, n, sgn):
    d, k, tau, zh, cs, uin = interlaced_cauchy(n, rows, 40 + n, rho_sign=sgn)
    want = O.cauchy_apply_explicit(uin, d, k, tau, zh, cs)
    plan = P.Plan(max(rows, n), max(rows, n), flags=P.FORCE_DIRECT)
    out, used = plan.cauchy_apply(T(uin), T(d), T(k, torch.int32), T(tau), T(zh), T(cs))
    assert not used
    E = _abs_scale(uin, d, k, tau, zh, cs)
    assert np.max(np.abs(N(out) - want) / E) <= 1e-13


@pytest.mark.parametrize("rows,n,sgn,eps", [(100, 65, 1.0, 1e-10), (257, 777, -1.0, 1e-10),
                                            (64, 2500, 1.0, 1e-10), (70, 3000, 1.0, 5.0 ** -20)])
def test_cauchy_apply_fmm(rows, n, sgn, eps):
    """Q23: FMM vs the explicit product within 10 eps of the per-entry error scale."""
    d, k, tau, zh, cs, uin = interlaced_cauchy(n, rows, 70 + n, rho_sign=sgn)
    want = O.cauchy_apply_explicit(uin, d, k, tau, zh, cs)
    plan = P.Plan(max(rows, n), max(rows, n), eps=eps, flags=P.FORCE_FMM)
    out, used = plan.cauchy_apply(T(uin), T(d), T(k, torch.int32), T(tau), T(zh), T(cs))
    assert used
    E = _abs_scale(uin, d, k, tau, zh, cs)
    assert np.max(np.abs(N(out) - want) / E) <= 10 * max(eps, 1e-13)


@pytest.mark.parametrize("n,sgn", [(3000, 1.0), (3000, -1.0)])
def test_cauchy_apply_fmm_one_sided(n, sgn):
    """Graded sources (C3's spectrum shape, d = 10^(-12 i / n)): the tree's leaves have
    geometrically varying widths, so the plan uses one-sided P2L / M2P terms (DESIGN.md
    §4.4; checked through the host planner) -- the FMM apply stays within Q23's bound."""
    from paper_1707_08369_b200._lib import fmm_tree_stats
    rng = np.random.default_rng(90 + n)
    d = np.sort(10.0 ** (-12.0 * np.arange(n) / n))
    gaps = np.diff(d)
    frac = rng.uniform(0.05, 0.95, size=n)
    k = np.arange(n, dtype=np.int32)
    tau = np.empty(n)
    if sgn > 0:
        tau[:-1] = frac[:-1] * gaps
        tau[-1] = frac[-1] * gaps[-1]
    else:
        tau[1:] = -frac[1:] * gaps
        tau[0] = -frac[0] * d[0]
    zh = rng.standard_normal(n)
    cs = rng.uniform(0.5, 2.0, size=n)
    uin = rng.standard_normal((96, n))
    st = fmm_tree_stats(d, k, tau, 1e-10)
    assert st["max_near"] <= 4, st  # the symmetric lists reach 5 leaves here (634 near pairs vs 382-384)
    want = O.cauchy_apply_explicit(uin, d, k, tau, zh, cs)
    plan = P.Plan(n, n, eps=1e-10, flags=P.FORCE_FMM)
    out, used = plan.cauchy_apply(T(uin), T(d), T(k, torch.int32), T(tau), T(zh), T(cs))
    assert used
    E = _abs_scale(uin, d, k, tau, zh, cs)
    assert np.max(np.abs(N(out) - want) / E) <= 10 * 1e-10


# ------------------------------------------------------------------ full update
def _gpu_update(U, s, V, a, b, **kw):
    Ug, sg, Vg = T(U), T(s), T(V)
    plan = P.Plan(U.shape[0], V.shape[0], **kw)
    rep = plan.update(Ug, sg, Vg, T(a), T(b))
    return Ug, sg, Vg, rep


def _check_update(U, s, V, a, b, flags=0, fmm_min_n=0):
    m, n = U.shape[0], V.shape[0]
    ref = O.svd_update(U, s, V, a, b)
    Ug, sg, Vg, rep = _gpu_update(U, s, V, a, b, flags=flags, fmm_min_n=fmm_min_n)
    A_hat = T((U * s[None, :]) @ V[:, :m].T + np.outer(a, b))
    res = float(torch.linalg.norm(A_hat @ Vg[:, :m] - Ug * sg[None, :], dim=0).max() / sg[0])
    I_m = torch.eye(m, dtype=torch.float64, device=DEV)
    I_n = torch.eye(n, dtype=torch.float64, device=DEV)
    orth = max(float((Ug.T @ Ug - I_m).abs().max()), float((Vg.T @ Vg - I_n).abs().max()))
    se = sigma_errors(N(sg), ref["sigma"])
    eu = vector_error(N(Ug), ref["U"], ref["sigma"] ** 2)
    ev = vector_error(N(Vg), ref["V"], ref["info"]["Dv_hat"])
    return dict(sigma=se, res=res, orth=orth, U=eu, V=ev, rep=rep)


@pytest.mark.parametrize("cfg,m,n,flags", [
    (1, None, None, 0),                      # C1 full size (direct path)
    (2, 256, 256, P.FORCE_FMM),              # C2 recipe, FMM path
    (2, 300, 300, P.FORCE_DIRECT),
    (3, 256, 256, P.FORCE_FMM),              # C3 graded recipe
    (4, 40, 160, 0),                         # C4 recipe: rectangular, null-space Householder
    (5, 200, 200, P.FORCE_FMM),              # C5 recipe: duplicated sigma
])
def test_update_parity(cfg, m, n, flags):
    inp = config_inputs(cfg, m=m, n=n, updates=1)
    a, b = inp["ab"][0]
    r = _check_update(inp["U"], inp["sigma"], inp["V"], a, b, flags=flags)
    assert_parity(f"update_parity C{cfg} {m}x{n} flags={flags}", r)


def test_update_noop_and_errors():
    inp = config_inputs(1, m=16, n=24, updates=1)
    U, s, V = inp["U"], inp["sigma"], inp["V"]
    Ug, sg, Vg, rep = _gpu_update(U, s, V, np.zeros(16), inp["ab"][0][1])
    assert rep["noop"] == 1 and np.array_equal(N(Ug), U) and np.array_equal(N(sg), s)
    b = inp["ab"][0][1].copy()
    b[3] = np.nan
    with pytest.raises(P.SVD1Error) as e:
        _gpu_update(U, s, V, inp["ab"][0][0], b)
    assert e.value.code == 2


def test_update_stream_c3_small():
    """Four chained updates on the C3 recipe: invariants hold through the stream
    (Q30: one-step parity at each step, oracle fed the GPU's previous factors)."""
    inp = config_inputs(3, m=192, n=192, updates=4)
    U, s, V = inp["U"], inp["sigma"], inp["V"]
    A = (U * s[None, :]) @ V.T
    Ug, sg, Vg = T(U), T(s), T(V)
    plan = P.Plan(192, 192, flags=P.FORCE_FMM)
    for (a, b) in inp["ab"]:
        Uprev, sprev, Vprev = N(Ug), N(sg), N(Vg)
        ref = O.svd_update(Uprev, sprev, Vprev, a, b)
        plan.update(Ug, sg, Vg, T(a), T(b))
        A = A + np.outer(a, b)
        e = sigma_errors(N(sg), ref["sigma"])
        At = T(A)
        res = float(torch.linalg.norm(At @ Vg - Ug * sg[None, :], dim=0).max() / sg[0])
        eu = vector_error(N(Ug), ref["U"], ref["sigma"] ** 2)
        ev = vector_error(N(Vg), ref["V"], ref["info"]["Dv_hat"])
        assert_parity("stream_c3_small step", dict(sigma=e, U=eu, V=ev, res=res))


@pytest.mark.parametrize("n,flags", [(24, 0), (600, P.FORCE_FMM)])
def test_repeated_sigma_pairing(n, flags):
    """Multiplicity-4 singular value -> multiplicity 2 after the update: the GPU's
    probe-based k x k pairing rotation (D5) gives a paired SVD (residual), and the
    cluster's subspaces match the oracle's."""
    rng = np.random.default_rng(n)
    s = np.sort(rng.uniform(1, 10, n))[::-1].copy()
    s[5:9] = s[5]
    U = np.linalg.qr(rng.standard_normal((n, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    r = _check_update(U, s, V, a, b, flags=flags)
    assert r["rep"]["pair_rotations"] >= 1
    assert r["res"] <= 1e-10 and r["orth"] <= 1e-10, r
    assert r["U"]["cluster"] <= 1e-9 and r["V"]["cluster"] <= 1e-9, r


# ------------------------------------------------------- FMM secular solve (§8(f) #2)
@pytest.fixture(scope="module")
def plan_secfmm():
    p = P.Plan(4096, 4096, eps=1e-10, flags=P.SECULAR_FMM)
    yield p
    p.close()


@pytest.mark.parametrize("n,kind,sgn", [(n, k, s) for n in (97, 700, 3000) for k in ("gaussian", "graded", "uniform")
                                         for s in (1.0, -1.0)])
def test_secular_fmm_parity(plan_secfmm, n, kind, sgn):
    """Roots with the far field of w from the secular FMM (near sources direct) agree with
    the bisection oracle as the direct solver does, and lie in w's rounding band."""
    rng = np.random.default_rng(n * 11 + len(kind))
    d, z, rho = random_secular(n, rng, kind=kind)
    rho = sgn * abs(rho)
    dfl = O.deflate(d, z, rho)
    d, z = dfl.d[dfl.active], dfl.z[dfl.active]
    n = d.size
    ko, to = O.secular_roots_bisect(d, z, rho)
    kg, tg, iters = plan_secfmm.secular_solve(T(d), T(z), rho)
    kg, tg = N(kg).astype(np.int64), N(tg)
    diff = ((d[kg] - d[ko]) + tg) - to
    scale = np.minimum(np.abs(to), np.abs(tg))
    assert np.max(np.abs(diff) / scale) <= 2e-12, (np.max(np.abs(diff) / scale), iters)
    w = O.secular_w(d, z, rho, kg, tg)
    terms = np.abs(z[None, :] ** 2 / ((d[None, :] - d[kg][:, None]) - tg[:, None]))
    assert np.all(np.abs(w) <= 64 * n * O.EPS * (1 + abs(rho) * terms.sum(axis=1)))
    assert iters <= 40


@pytest.mark.parametrize("cfg,m,n", [(3, 512, 512), (5, 600, 600), (4, 256, 1024)])
def test_update_parity_secular_fmm(cfg, m, n):
    """Whole updates with every secular solve on the FMM path (D2-D4 tolerances)."""
    inp = config_inputs(cfg, m=m, n=n, updates=1)
    a, b = inp["ab"][0]
    r = _check_update(inp["U"], inp["sigma"], inp["V"], a, b, flags=P.SECULAR_FMM)
    assert r["rep"]["n_active"][0] > 64  # the FMM secular solve ran (sizes > 64)
    assert_parity(f"update_parity_secular_fmm C{cfg} {m}x{n}", r)


def test_rectangular_stream_null_root():
    """C4 recipe (m < n), five chained updates: the V side's null-space root lands on
    mu = 0 exactly, where a padded source of the direct apply (d = 0) once gave 0/0."""
    inp = config_inputs(4, m=64, n=256, updates=5)
    Ug, sg, Vg = T(inp["U"]), T(inp["sigma"]), T(inp["V"])
    plan = P.Plan(64, 256)
    A = (inp["U"] * inp["sigma"][None, :]) @ inp["V"][:, :64].T
    for a, b in inp["ab"]:
        plan.update(Ug, sg, Vg, T(a), T(b))
        A = A + np.outer(a, b)
    assert bool(torch.isfinite(Vg).all()) and bool(torch.isfinite(Ug).all())
    res = float(torch.linalg.norm(T(A) @ Vg[:, :64] - Ug * sg[None, :], dim=0).max() / sg[0])
    assert res <= 1e-10
