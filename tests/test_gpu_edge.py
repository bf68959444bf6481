"""Degenerate whole updates on the CUDA path (synth/edge.py), through the C ABI, against
the oracle (Alg 6.1) at the north star's tolerances (readings D2-D4): the
smallest shapes (1x1 .. 3x3, 1x3, 2x5), update vectors inside a few singular directions
(zero weights), rank-deficient and fully repeated spectra, A and a b^T scaled
by 1e80 / 1e-20, updates 1e-11 and 1e9 times ||A||, and an unbalanced a b^T = (1e8 a)(1e-8 b)^T
(reading D9: the per-side power-of-two balance before the Schur split), a
downdate to an exact zero singular value, A = 0, a one-entry change and b in the null space
of A's rows.  Also:
(2^t a, b / 2^t) gives bitwise the same factors (D9), and a pipelined stream with unbalanced
and extreme-scale updates matches the per-update path."""
import math

import numpy as np
import pytest

import oracle as O
from compare import assert_parity, sigma_errors, vector_error
from synth import EDGE_CASES, EDGE_RES_TOL, edge_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1707_08369_b200 as P  # noqa: E402

DEV = torch.device("cuda:0")


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, torch.float64)


def N(x):
    return x.detach().cpu().numpy()


def _gpu(U, s, V, a, b, flags=0):
    Ug, sg, Vg = T(U), T(s), T(V)
    plan = P.Plan(U.shape[0], V.shape[0], flags=flags)
    rep = plan.update(Ug, sg, Vg, T(a), T(b))
    torch.cuda.synchronize()
    plan.close()
    return Ug, sg, Vg, rep


@pytest.mark.parametrize("flags", [0, P.FORCE_FMM])
@pytest.mark.parametrize("name", EDGE_CASES)
def test_edge_update_parity(name, flags):
    U, s, V, a, b = edge_case(name)
    m, n = U.shape[0], V.shape[0]
    if flags and m < 8:
        pytest.skip("FMM apply needs more than a handful of points")
    ref = O.svd_update(U, s, V, a, b)
    Ug, sg, Vg, rep = _gpu(U, s, V, a, b, flags)
    A_hat = (U * s[None, :]) @ V[:, :m].T + np.outer(a, b)
    f = math.ldexp(1.0, math.frexp(float(np.max(np.abs(A_hat))))[1])  # exact rescaling for the
    Ah = T(A_hat / f)                                                  # residual (1e80 / 1e-20)
    res = float(torch.linalg.norm(Ah @ Vg[:, :m] - Ug * (sg / f)[None, :], dim=0).max() / (sg[0] / f))
    orth = max(float((Ug.T @ Ug - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max()),
               float((Vg.T @ Vg - torch.eye(n, dtype=torch.float64, device=DEV)).abs().max()))
    r = dict(sigma=sigma_errors(N(sg), ref["sigma"]), res=res, orth=orth,
             U=vector_error(N(Ug), ref["U"], ref["sigma"] ** 2),
             V=vector_error(N(Vg), ref["V"], ref["info"]["Dv_hat"]))
    assert_parity(f"edge {name} flags={flags}", r, res_tol=EDGE_RES_TOL.get(name, 1e-10))


@pytest.mark.parametrize("name", ["tiny33", "a_in_span", "rank_deficient", "scaled_down", "unbalanced"])
def test_edge_balance_rescaling_bitwise(name):
    """D9 on the GPU: (2^t a, b / 2^t) gives bitwise the same factors."""
    U, s, V, a, b = edge_case(name)
    base = _gpu(U, s, V, a, b)
    for t in (-30, 7, 33):
        other = _gpu(U, s, V, a * 2.0 ** t, b / 2.0 ** t)
        for x, y in zip(base[:3], other[:3]):
            assert torch.equal(x, y), (name, t)


def test_edge_stream_matches_per_update():
    """A pipelined stream (svd1_update_batch) through unbalanced, tiny and huge updates:
    the same factors as the per-update path (singular values to 1e-12, columns gap-aware)."""
    U, s, V, _, _ = edge_case("unbalanced", m=96)
    rng = np.random.default_rng(77)
    m = n = 96
    ab = [(rng.standard_normal(m), rng.standard_normal(n)),
          (1e8 * rng.standard_normal(m), 1e-8 * rng.standard_normal(n)),
          (1e-12 * rng.standard_normal(m), rng.standard_normal(n)),
          (1e-3 * rng.standard_normal(m), 1e5 * rng.standard_normal(n)),
          (rng.standard_normal(m), rng.standard_normal(n))]
    outs = []
    for batch in (True, False):
        Ug, sg, Vg = T(U), T(s), T(V)
        plan = P.Plan(m, n, flags=P.FORCE_FMM)
        if batch:
            plan.update_batch(Ug, sg, Vg, T(np.stack([a for a, _ in ab])), T(np.stack([b for _, b in ab])))
        else:
            for a, b in ab:
                plan.update(Ug, sg, Vg, T(a), T(b))
        torch.cuda.synchronize()
        plan.close()
        outs.append((N(Ug), N(sg), N(Vg)))
    (Ub, sb, Vb), (Us, ss, Vs) = outs
    assert np.max(np.abs(sb - ss)) <= 1e-12 * ss[0]
    gu = vector_error(Ub, Us, ss ** 2)
    gv = vector_error(Vb[:, :m], Vs[:, :m], ss ** 2)
    assert max(gu["isolated"], gu["cluster"], gv["isolated"], gv["cluster"]) <= 1e-10, (gu, gv)
    A = (U * s[None, :]) @ V.T
    for a, b in ab:
        A = A + np.outer(a, b)
    res = np.max(np.linalg.norm(A @ Vb[:, :m] - Ub * sb[None, :], axis=0)) / sb[0]
    assert res <= 1e-10, res


def test_edge_stream_repeated_sigma():
    """A pipelined stream on A = 2 Q1 Q2^T (one singular value of multiplicity 48): every
    update leaves a cluster of 46, 44, 42 equal values paired from the tracked coordinates
    (D5 beyond the probes); the factors match the per-update path and the accumulated A."""
    U, s, V, _, _ = edge_case("all_equal")
    rng = np.random.default_rng(78)
    m = n = U.shape[0]
    ab = [(rng.standard_normal(m), rng.standard_normal(n)) for _ in range(3)]
    outs = []
    for batch in (True, False):
        Ug, sg, Vg = T(U), T(s), T(V)
        plan = P.Plan(m, n)
        if batch:
            reps = plan.update_batch(Ug, sg, Vg, T(np.stack([a for a, _ in ab])), T(np.stack([b for _, b in ab])))
        else:
            reps = [plan.update(Ug, sg, Vg, T(a), T(b)) for a, b in ab]
        torch.cuda.synchronize()
        plan.close()
        assert all(r["pair_rotations"] >= 1 for r in reps), [r["pair_rotations"] for r in reps]
        outs.append((N(Ug), N(sg), N(Vg)))
    (Ub, sb, Vb), (Us, ss, Vs) = outs
    assert np.max(np.abs(sb - ss)) <= 1e-12 * ss[0]
    A = (U * s[None, :]) @ V.T
    for a, b in ab:
        A = A + np.outer(a, b)
    for Uo, so, Vo in outs:
        res = np.max(np.linalg.norm(A @ Vo[:, :m] - Uo * so[None, :], axis=0)) / so[0]
        orth = max(np.max(np.abs(Uo.T @ Uo - np.eye(m))), np.max(np.abs(Vo.T @ Vo - np.eye(n))))
        assert res <= 1e-10 and orth <= 1e-10, (res, orth)
        e = sigma_errors(so, np.linalg.svd(A, compute_uv=False))
        assert e["gram"] <= 1e-12, e


def test_edge_cluster_beyond_tracking_refused():
    """A singular value repeated 300 times (> the 256 columns D5 tracks) is refused with
    SVD1_E_UNSUPPORTED before any write: the factors are left unchanged."""
    U, s, V, a, b = edge_case("all_equal", m=300)
    Ug, sg, Vg = T(U), T(s), T(V)
    plan = P.Plan(300, 300)
    with pytest.raises(P.SVD1Error) as e:
        plan.update(Ug, sg, Vg, T(a), T(b))
    torch.cuda.synchronize()
    plan.close()
    assert e.value.code == 9
    assert np.array_equal(N(Ug), U) and np.array_equal(N(sg), s) and np.array_equal(N(Vg), V)


@pytest.mark.parametrize("name,m", [("all_equal", 200), ("rank_deficient", 400), ("scaled_down", 600),
                                    ("unbalanced", 600), ("a_in_span", 500), ("downdate_top", 500)])
def test_edge_update_parity_fmm_sizes(name, m):
    """The same recipes at sizes where the forced FMM apply has a real tree (several levels,
    far-field and one-sided terms)."""
    U, s, V, a, b = edge_case(name, m=m)
    ref = O.svd_update(U, s, V, a, b)
    Ug, sg, Vg, rep = _gpu(U, s, V, a, b, P.FORCE_FMM)
    n = V.shape[0]
    A_hat = (U * s[None, :]) @ V[:, :m].T + np.outer(a, b)
    f = math.ldexp(1.0, math.frexp(float(np.max(np.abs(A_hat))))[1])
    Ah = T(A_hat / f)
    res = float(torch.linalg.norm(Ah @ Vg[:, :m] - Ug * (sg / f)[None, :], dim=0).max() / (sg[0] / f))
    orth = max(float((Ug.T @ Ug - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max()),
               float((Vg.T @ Vg - torch.eye(n, dtype=torch.float64, device=DEV)).abs().max()))
    r = dict(sigma=sigma_errors(N(sg), ref["sigma"]), res=res, orth=orth,
             U=vector_error(N(Ug), ref["U"], ref["sigma"] ** 2),
             V=vector_error(N(Vg), ref["V"], ref["info"]["Dv_hat"]))
    assert_parity(f"edge {name} m={m} FMM", r, res_tol=EDGE_RES_TOL.get(name, 1e-10))


@pytest.mark.parametrize("k", [3, 5, 10, 40])
def test_edge_near_equal_run(k):
    """k distinct singular values 4 ulp apart (not bitwise equal): runs of up to 6 are solved as
    distinct poles (the update splits them, or the probes pair what stays clustered); longer runs
    are taken as one repeated value (reading D10, a backward perturbation <= 64 eps ||A||), which
    deflates and is paired from the tracked coordinates (D5).  Nothing is left unpaired."""
    from synth import haar
    rng = np.random.default_rng(5 + k)
    m = n = 64
    sig = np.sort(rng.uniform(1, 10, m))[::-1].copy()
    sig[10:10 + k] = 5.0 * (1 + 4 * O.EPS * np.arange(k))[::-1]
    sig = np.sort(sig)[::-1].copy()  # (descending, as the API takes it)
    U, V = haar(m, rng), haar(n, rng)
    a, b = rng.standard_normal(m), rng.standard_normal(n)
    ref = O.svd_update(U, sig, V, a, b)
    Ug, sg, Vg, rep = _gpu(U, sig, V, a, b)
    A_hat = (U * sig[None, :]) @ V.T + np.outer(a, b)
    res = float(torch.linalg.norm(T(A_hat) @ Vg - Ug * sg[None, :], dim=0).max() / sg[0])
    orth = max(float((Ug.T @ Ug - torch.eye(m, dtype=torch.float64, device=DEV)).abs().max()),
               float((Vg.T @ Vg - torch.eye(n, dtype=torch.float64, device=DEV)).abs().max()))
    assert rep["unpaired_clusters"] == 0
    r = dict(sigma=sigma_errors(N(sg), ref["sigma"]), res=res, orth=orth,
             U=vector_error(N(Ug), ref["U"], ref["sigma"] ** 2),
             V=vector_error(N(Vg), ref["V"], ref["info"]["Dv_hat"]))
    assert_parity(f"edge near-equal run k={k}", r)


def test_graded_tail_not_reported_unpaired():
    """The graded C3 recipe's tail forms clusters under the absolute 64 eps sigma_1^2 rule, but
    its values are 0.7 % apart relative to themselves, so every column is fixed up to sign:
    none of them is reported as unpaired."""
    from synth import config_inputs
    inp = config_inputs(3, m=1024, n=1024, updates=4)
    Ug, sg, Vg = T(inp["U"]), T(inp["sigma"]), T(inp["V"])
    plan = P.Plan(1024, 1024)
    reps = plan.update_batch(Ug, sg, Vg, T(np.stack([a for a, _ in inp["ab"]])), T(np.stack([b for _, b in inp["ab"]])))
    torch.cuda.synchronize()
    plan.close()
    assert all(r["unpaired_clusters"] == 0 for r in reps), [r["unpaired_clusters"] for r in reps]
