"""Pins of the CPU oracle against things other than itself (`-m "not gpu"`).

Worked examples (tests/golden/*.json, each citing SPEC.md / PAPER.md), closed
forms, brute-force Jacobi eigen/SVD (tests/brute.py), LAPACK as a library
routine for the special case it computes, and invariants.  Chosen so that a
dropped term, wrong sign, wrong index or transposed operand in any oracle
function fails at least one test.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from brute import jacobi_eigvalsh, jacobi_svd
from compare import sigma_errors, vector_error
from synth import gaussian_factors, graded_factors, paper_uniform, random_secular, config_inputs, EDGE_CASES, EDGE_RES_TOL, edge_case

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ Schur 2x2
def test_schur_golden():
    for c in gold("schur_2x2.json")["cases"]:
        r1, r2, Q = O.schur_sym_2x2(np.array(c["M"], float))
        assert r1 == pytest.approx(c["rho1"], abs=1e-15)
        assert r2 == pytest.approx(c["rho2"], abs=1e-15)
        M = np.array(c["M"], float)
        assert np.max(np.abs(Q @ np.diag([r1, r2]) @ Q.T - M)) <= 1e-14


def test_schur_random_reconstruction():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        x = rng.standard_normal(3) * 10.0 ** rng.uniform(-3, 3)
        M = np.array([[x[0], x[1]], [x[1], x[2]]])
        r1, r2, Q = O.schur_sym_2x2(M)
        assert r1 >= r2
        assert np.max(np.abs(Q @ Q.T - np.eye(2))) <= 1e-14
        assert np.max(np.abs(Q @ np.diag([r1, r2]) @ Q.T - M)) <= 1e-13 * (1 + np.max(np.abs(M)))


@pytest.mark.parametrize("beta", [0.0, 1e-8, 0.5, 1.0, 37.0, 4096.0, 1e12])
def test_schur_update_split(beta):
    """[[beta,1],[1,0]]: rho1 rho2 = det = -1, rho1 + rho2 = beta."""
    r1, r2, Q = O.schur_update_2x2(beta)
    assert r1 > 0 > r2
    assert r1 * r2 == pytest.approx(-1.0, rel=1e-15)
    assert r1 + r2 == pytest.approx(beta, rel=1e-14, abs=1e-15)


# ----------------------------------------------------------------- STEP 1
def test_prepare_identity_golden():
    g = gold("svd_update.json")["prepare_identity"]
    ing = O.prepare_update(np.array(g["U"], float), np.array(g["sigma"], float),
                           np.array(g["V"], float), np.array(g["a"], float), np.array(g["b"], float))
    assert np.array_equal(ing["b_tilde"], np.array(g["b_tilde"], float))
    assert np.array_equal(ing["a_tilde"], np.array(g["a_tilde"], float))
    assert ing["beta"] == g["beta"] and ing["alpha"] == g["alpha"]


def test_prepare_bruteforce():
    """random 3x4 case equals brute-force evaluation of the products."""
    rng = np.random.default_rng(2)
    m, n = 3, 4
    U, s, V = gaussian_factors(m, n, rng)
    a, b = rng.standard_normal(m), rng.standard_normal(n)
    A = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            A[i, j] = sum(U[i, k] * s[k] * V[j, k] for k in range(m))
    bt = [sum(A[i, j] * b[j] for j in range(n)) for i in range(m)]
    at = [sum(A[i, j] * a[i] for i in range(m)) for j in range(n)]
    ing = O.prepare_update(U, s, V, a, b)
    assert np.max(np.abs(ing["b_tilde"] - bt)) <= 1e-14
    assert np.max(np.abs(ing["a_tilde"] - at)) <= 1e-14
    assert np.array_equal(ing["Dv"][m:], np.zeros(n - m))


# ------------------------------------------------------------ secular solver
def test_secular_eval_golden():
    for c in gold("secular.json")["eval"]:
        d = np.array(c["d"])
        w = O.secular_w(d, np.array(c["z"]), c["rho"], np.array([0]), np.array([c["mu"] - d[0]]))
        assert w[0] == pytest.approx(c["w"], abs=1e-15)


def test_secular_roots_golden():
    for c in gold("secular.json")["roots"]:
        d = np.array(c["d"])
        k, tau = O.secular_roots_bisect(d, np.array(c["z"]), c["rho"])
        mu = d[k] + tau
        assert np.max(np.abs(mu - np.array(c["mu"]))) <= 4e-16 * max(1.0, np.max(np.abs(mu)))


@pytest.mark.parametrize("seed", range(40))
def test_secular_vs_dense_eigensolvers(seed):
    """roots equal the eigenvalues of D + rho z z^T computed by a
    brute-force Jacobi eigensolver and by LAPACK (special case = library routine)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 40))
    d, z, rho = random_secular(n, rng, kind=["gaussian", "uniform", "graded"][seed % 3])
    dfl = O.deflate(d, z, rho)
    assert dfl.active.size == n  # random data: nothing deflates
    k, tau = O.secular_roots_bisect(d, z, rho)
    mu = d[k] + tau
    B = np.diag(d) + rho * np.outer(z, z)
    nb = np.max(np.abs(np.linalg.eigvalsh(B)))
    assert np.max(np.abs(mu - np.linalg.eigvalsh(B))) <= 1e-13 * nb
    if n <= 24:
        assert np.max(np.abs(mu - jacobi_eigvalsh(B))) <= 1e-12 * nb


@pytest.mark.parametrize("seed", range(60))
def test_secular_interlacing_and_trace(seed):
    """S:134/S:142 strict interlacing; S:143 trace conservation."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 129))
    d, z, rho = random_secular(n, rng, kind=["gaussian", "uniform", "graded"][seed % 3],
                               n_zero=int(rng.integers(0, 3)), n_dup=int(rng.integers(0, 3)))
    dfl = O.deflate(d, z, rho)
    da, za = dfl.d[dfl.active], dfl.z[dfl.active]
    assert np.all(np.diff(da) > 0)
    k, tau = O.secular_roots_bisect(da, za, rho)
    mu = da[k] + tau
    assert np.all(np.diff(mu) > 0)
    if rho > 0:
        assert np.all(mu > da) and np.all(mu[:-1] < da[1:])
        assert mu[-1] <= da[-1] + rho * float(za @ za) * (1 + 1e-15)
    else:
        assert np.all(mu < da) and np.all(mu[1:] > da[:-1])
        assert mu[0] >= da[0] + rho * float(za @ za) * (1 + 1e-15)
    total = float(np.sum(mu) + np.sum(dfl.d[dfl.deflated]))
    scale = float(np.sum(np.abs(d)) + abs(rho) * float(z @ z))
    assert abs(total - (float(np.sum(d)) + rho * float(z @ z))) <= 1e-13 * scale
    w = O.secular_w(da, za, rho, k, tau)
    # |w| at the root is within the rounding band of its evaluation
    terms = np.abs(za[None, :] ** 2 / ((da[None, :] - da[k][:, None]) - tau[:, None]))
    band = 1 + abs(rho) * terms.sum(axis=1)
    assert np.all(np.abs(w) <= 64 * n * O.EPS * band)


# ----------------------------------------------------------------- deflation
def test_deflation_golden():
    for c in gold("deflation.json")["cases"]:
        dfl = O.deflate(np.array(c["d"]), np.array(c["z"]), c["rho"])
        assert dfl.active.size == c["n_active"]
        assert np.allclose(dfl.d[dfl.deflated], c["deflated_eigs"], atol=0)
        if "carried_weight_abs" in c:
            assert abs(dfl.z[dfl.active[0]]) == pytest.approx(c["carried_weight_abs"], abs=1e-15)


@pytest.mark.parametrize("seed", range(20))
def test_deflation_preserves_spectrum_and_is_idempotent(seed):
    """S:145 idempotence; deflated problem has the same eigenvalues (dense
    eigensolver, library routine on the undeflated and deflated matrices)."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(4, 60))
    d, z, rho = random_secular(n, rng, kind="uniform", n_zero=int(rng.integers(1, 4)),
                               n_dup=int(rng.integers(1, 6)))
    dfl = O.deflate(d, z, rho)
    assert dfl.deflated.size >= 1
    B = np.diag(d) + rho * np.outer(z, z)
    B2 = np.diag(dfl.d) + rho * np.outer(dfl.z, dfl.z)
    e1, e2 = np.linalg.eigvalsh(B), np.linalg.eigvalsh(B2)
    assert np.max(np.abs(e1 - e2)) <= 1e-12 * np.max(np.abs(e1))
    # orthogonal transform: the rotated basis reproduces B
    Q = np.eye(n)
    from oracle.svd1_oracle import _apply_ops_cols
    _apply_ops_cols(dfl.ops, Q)
    assert np.max(np.abs(Q @ B2 @ Q.T - B)) <= 1e-12 * np.max(np.abs(B))
    da, za = dfl.d[dfl.active], dfl.z[dfl.active]
    again = O.deflate(da, za, rho)
    assert again.deflated.size == 0 and np.array_equal(again.z, za)


# ------------------------------------------------------------------- Loewner
@pytest.mark.parametrize("seed", range(12))
def test_loewner_identities(seed):
    rng = np.random.default_rng(1300 + seed)
    n = int(rng.integers(2, 200))
    d, z, rho = random_secular(n, rng, kind=["gaussian", "graded", "uniform"][seed % 3])
    k, tau = O.secular_roots_bisect(d, z, rho)
    zh = O.loewner_zhat(d, k, tau, rho, z)
    mu = d[k] + tau
    # trace identity ||zhat||^2 = (sum mu - sum d) / rho  (characteristic polynomial)
    lhs = float(zh @ zh)
    rhs = float(np.sum(tau + (d[k] - d))) / rho
    assert lhs == pytest.approx(rhs, rel=1e-11)
    assert np.max(np.abs(zh / z - 1)) <= 1e-10
    assert np.all(np.sign(zh) == np.sign(z))
    # mu are roots of the zhat secular equation
    w = O.secular_w(d, zh, rho, k, tau)
    terms = np.abs(zh[None, :] ** 2 / ((d[None, :] - d[k][:, None]) - tau[:, None]))
    assert np.all(np.abs(w) <= 1e-11 * (1 + abs(rho) * terms.sum(axis=1)))
    assert np.all(np.diff(mu) > 0)


# ------------------------------------------------------------- Cauchy / X
def test_cauchy_golden():
    g = gold("cauchy.json")
    lam, mu = np.array(g["build"]["lambda"]), np.array(g["build"]["mu"])
    # gap form with origin 0: mu_j = lam_0 + (mu_j - lam_0)
    k = np.zeros(2, np.int64)
    tau = mu - lam[0]
    C = O.cauchy_apply_explicit(np.eye(2), lam, k, tau, np.ones(2), np.ones(2))
    assert np.max(np.abs(C - np.array(g["build"]["C"]))) <= 1e-15
    u = np.array(g["matvec"]["u"])[None, :]
    f = O.cauchy_apply_explicit(u, lam, k, tau, np.ones(2), np.ones(2))
    assert np.max(np.abs(f[0] - np.array(g["matvec"]["f"]))) <= 1e-15
    c = g["colnorm"]
    lam2 = np.array(c["lambda"])
    X, cn = O.cauchy_X(lam2, np.array([0]), np.array(c["mu"]) - lam2[0], np.array(c["abar"]))
    assert cn[0] == pytest.approx(c["norm"], abs=1e-15)


def test_eigvec_n2_golden():
    g = gold("cauchy.json")["eigvec_n2"]
    d, z = np.array(g["d"]), np.array(g["z"])
    U, D = O.sym_rank_one_eig(np.eye(2), d, z, g["rho"])
    assert np.max(np.abs(np.abs(U) - np.array(g["vectors_abs"]))) <= 1e-15
    assert np.max(np.abs(D - np.array([1 - math.sqrt(2) / 2, 1 + math.sqrt(2) / 2]))) <= 4e-16


@pytest.mark.parametrize("seed", range(10))
def test_X_orthogonal_and_diagonalises(seed):
    """C~ orthogonal (P:188 'to make the final matrix orthogonal') and
    X diag(mu) X^T = D + rho zhat zhat^T (P:87 Eq. BTildeCDC1)."""
    rng = np.random.default_rng(1500 + seed)
    n = int(rng.integers(2, 120))
    d, z, rho = random_secular(n, rng, kind=["gaussian", "graded", "uniform"][seed % 3])
    k, tau = O.secular_roots_bisect(d, z, rho)
    zh = O.loewner_zhat(d, k, tau, rho, z)
    X, _ = O.cauchy_X(d, k, tau, zh)
    mu = d[k] + tau
    assert np.max(np.abs(X.T @ X - np.eye(n))) <= 1e-13
    B = np.diag(d) + rho * np.outer(zh, zh)
    assert np.max(np.abs(X @ np.diag(mu) @ X.T - B)) <= 1e-13 * np.max(np.abs(B))


def test_rank_one_update_reconstruction():
    """U_new diag(D_new) U_new^T = U D U^T + rho a1 a1^T."""
    rng = np.random.default_rng(7)
    n = 32
    U = np.linalg.qr(rng.standard_normal((n, n)))[0]
    D = rng.standard_normal(n)
    a1 = rng.standard_normal(n)
    for rho in (2.5, -0.7):
        Un, Dn = O.sym_rank_one_eig(U, D, a1, rho)
        lhs = (Un * Dn[None, :]) @ Un.T
        rhs = (U * D[None, :]) @ U.T + rho * np.outer(a1, a1)
        assert np.max(np.abs(lhs - rhs)) <= 1e-13 * np.max(np.abs(rhs))
        assert O.orth_defect(Un) <= 1e-13
        assert np.all(np.diff(Dn) >= 0)


def test_orth_defect_golden():
    for c in gold("orth_defect.json")["cases"]:
        assert O.orth_defect(np.array(c["M"], float)) == pytest.approx(c["defect"], abs=c["tol"] + 1e-300)


# --------------------------------------------------------------- Alg 6.1
def test_svd_update_identity_golden():
    g = gold("svd_update.json")["identity_update"]
    r = O.svd_update(np.array(g["U"], float), np.array(g["sigma"], float), np.array(g["V"], float),
                     np.array(g["a"], float), np.array(g["b"], float))
    assert np.max(np.abs(r["sigma"] - np.array(g["sigma_hat"]))) <= 2 * O.EPS * 2.0  # 2 ulp of 2
    A = np.diag(g["sigma_hat"])
    assert np.max(np.abs((r["U"] * r["sigma"]) @ r["V"].T - A)) <= 1e-15


def test_svd_update_noop():
    """O1 / S:467 / S:503: a = 0 or b = 0 leaves the factors unchanged."""
    rng = np.random.default_rng(3)
    U, s, V = gaussian_factors(6, 9, rng)
    r = O.svd_update(U, s, V, np.zeros(6), rng.standard_normal(9))
    assert np.array_equal(r["U"], U) and np.array_equal(r["sigma"], s) and np.array_equal(r["V"], V)


@pytest.mark.parametrize("mn", [(2, 2), (5, 5), (8, 13), (16, 16), (24, 40), (32, 32)])
def test_svd_update_vs_brute_force_jacobi(mn):
    """North star: the oracle checked against a brute-force one-sided-Jacobi
    SVD of A_hat, plus orthogonality and residual."""
    m, n = mn
    rng = np.random.default_rng(11 * m + n)
    U, s, V = gaussian_factors(m, n, rng)
    a, b = rng.standard_normal(m), rng.standard_normal(n)
    r = O.svd_update(U, s, V, a, b)
    A_hat = (U * s) @ V[:, :m].T + np.outer(a, b)
    Qj, sj, Vj = jacobi_svd(A_hat)
    e = sigma_errors(r["sigma"], sj)
    assert e["gram"] <= 1e-13 and e["rel_top"] <= 1e-12
    assert O.orth_defect(r["U"]) <= 1e-13 and O.orth_defect(r["V"]) <= 1e-13
    assert O.column_residual(A_hat, r["U"], r["sigma"], r["V"]) <= 1e-13
    ve = vector_error(r["U"], Qj, sj ** 2)
    assert ve["isolated"] <= 1e-10 and ve["cluster"] <= 1e-10
    ve = vector_error(r["V"][:, :m], Vj, sj ** 2)
    assert ve["isolated"] <= 1e-10 and ve["cluster"] <= 1e-10


@pytest.mark.parametrize("kind", ["gaussian", "graded", "dup", "rect_small"])
def test_svd_update_invariants(kind):
    """Weyl interlacing of singular values under a rank-one change, Frobenius
    identity sum s_hat^2 = sum s^2 + 2 x_a^T Sigma y_b + alpha beta, residual,
    orthogonality, left/right eigenvalue consistency."""
    rng = np.random.default_rng({"gaussian": 1, "graded": 2, "dup": 3, "rect_small": 4}[kind])
    if kind == "gaussian":
        U, s, V = gaussian_factors(48, 48, rng)
        a, b = rng.standard_normal(48), rng.standard_normal(48)
    elif kind == "graded":
        U, s, V = graded_factors(96, rng)
        a, b = rng.standard_normal(96), rng.standard_normal(96)
    elif kind == "dup":
        inp = config_inputs(5, m=80, n=80, updates=1)
        U, s, V = inp["U"], inp["sigma"], inp["V"]
        a, b = inp["ab"][0]
    else:
        inp = config_inputs(4, m=24, n=96, updates=1)
        U, s, V = inp["U"], inp["sigma"], inp["V"]
        a, b = inp["ab"][0]
    m = U.shape[0]
    r = O.svd_update(U, s, V, a, b)
    sh = r["sigma"]
    tol = 1e-13 * sh[0]
    assert np.all(sh[1:] <= s[:-1] + tol) and np.all(s[1:] <= sh[:-1] + tol)
    xa, yb = U.T @ a, V.T @ b
    frob = float(np.sum(s ** 2) + 2 * xa @ (s * yb[:m]) + (a @ a) * (b @ b))
    assert float(np.sum(sh ** 2)) == pytest.approx(frob, rel=1e-12)
    A_hat = (U * s) @ V[:, :m].T + np.outer(a, b)
    assert O.column_residual(A_hat, r["U"], sh, r["V"]) <= 1e-12
    assert O.orth_defect(r["U"]) <= 1e-12 and O.orth_defect(r["V"]) <= 1e-12
    dv = r["info"]["Dv_hat"][:m]
    assert np.max(np.abs(dv - r["info"]["D_hat"])) <= 1e-12 * dv[0]
    sv = np.linalg.svd(A_hat, compute_uv=False)
    e = sigma_errors(sh, sv)
    assert e["gram"] <= 1e-13 and e["rel_top"] <= 1e-12


def test_table2_analogue():
    """PAPER.md:456-470 Table 2: Error (Eq. error) on square matrices
    with entries in [1,9].  The paper's values are a ceiling; a correct
    method is far below them."""
    for row in gold("paper_table2.json")["rows"]:
        n = row["n"]
        A, a, b = paper_uniform(n, n, 4000 + n)
        U, s, Vt = np.linalg.svd(A)
        r = O.svd_update(U, s, Vt.T, a, b)
        A_hat = A + np.outer(a, b)
        err = O.paper_error(A_hat, r["U"], r["sigma"], r["V"])
        assert err < row["error"]
        assert err <= 1e-13


def test_probe_sign_rule_matches_explicit():
    """Q11: the small-vector probe rule picks the same signs as u_i^T A_hat v_i."""
    rng = np.random.default_rng(21)
    for (m, n) in [(12, 12), (20, 33), (40, 40)]:
        U, s, V = gaussian_factors(m, n, rng)
        a, b = rng.standard_normal(m), rng.standard_normal(n)
        r1 = O.svd_update(U, s, V, a, b, sign_rule="explicit")
        r2 = O.svd_update(U, s, V, a, b, sign_rule="probe")
        assert np.array_equal(r1["U"], r2["U"])
        assert np.max(np.abs(r1["V"][:, :m] - r2["V"][:, :m])) == 0.0


def test_large_mode_rows_match_full():
    """O8: sampled rows with the chained z (B7) agree with the literal full
    computation on those rows (rows are independent)."""
    rng = np.random.default_rng(31)
    m, n = 40, 56
    U, s, V = gaussian_factors(m, n, rng)
    a, b = rng.standard_normal(m), rng.standard_normal(n)
    r1 = O.svd_update(U, s, V, a, b, sign_rule="probe")
    ru, rv = np.arange(0, m, 3), np.arange(1, n, 4)
    r2 = O.svd_update(U, s, V, a, b, sign_rule="probe", rows=(ru, rv))
    assert np.max(np.abs(r2["sigma"] - r1["sigma"])) <= 1e-14 * r1["sigma"][0]
    assert np.max(np.abs(r2["U"] - r1["U"][ru])) <= 1e-12
    assert np.max(np.abs(r2["V"][:, :m] - r1["V"][rv][:, :m])) <= 1e-12


@pytest.mark.parametrize("rule", ["explicit", "probe"])
def test_repeated_singular_values_are_paired(rule):
    """A singular value of multiplicity 4 in A keeps multiplicity 2 after the two
    symmetric rank-1 updates of each side; the U and V bases of that subspace come
    out independently, so a sign flip cannot pair them (D5): the k x k pairing
    rotation must, or the residual is O(sigma).  Checked against the residual and a
    brute-force Jacobi SVD."""
    rng = np.random.default_rng(8)
    m = n = 24
    s = np.sort(rng.uniform(1, 10, n))[::-1].copy()
    s[5:9] = s[5]  # multiplicity 4
    U = np.linalg.qr(rng.standard_normal((m, m)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    a, b = rng.standard_normal(m), rng.standard_normal(n)
    r = O.svd_update(U, s, V, a, b, sign_rule=rule)
    A_hat = (U * s) @ V.T + np.outer(a, b)
    assert r["info"]["rotations"] >= 1
    assert O.column_residual(A_hat, r["U"], r["sigma"], r["V"]) <= 1e-13
    assert O.orth_defect(r["V"]) <= 1e-13
    _, sj, _ = jacobi_svd(A_hat)
    assert sigma_errors(r["sigma"], sj)["gram"] <= 1e-13


# ------------------------------------------------------------------ metrics
def test_paper_error_hand_cases():
    """paper_error (Q24: the denominator is the largest singular value of A_hat)
    on hand-computed 2x2 / 2x3 cases: a transposed V, a Frobenius-norm denominator or a
    sum instead of a max would each change one of these values."""
    A = np.array([[3.0, 0.0], [0.0, 4.0]])      # ||A||_2 = 4 (Frobenius 5)
    Us = np.array([[0.0, 1.0], [1.0, 0.0]])     # u1 = e2, u2 = e1
    assert O.paper_error(A, Us, np.array([4.0, 3.0]), Us) == 0.0
    # sigma_2 off by 0.5 -> residual 0.5 at entry (0, 0): error 0.5 / 4
    assert O.paper_error(A, Us, np.array([4.0, 2.5]), Us) == pytest.approx(0.125, rel=1e-15)
    # both off: max (not sum) of |R| = 0.5, not 0.5 + 0.25
    assert O.paper_error(A, Us, np.array([3.75, 2.5]), Us) == pytest.approx(0.125, rel=1e-15)
    # rectangular m = 2 < n = 3: A_hat = 5 e1 e3^T, sigma = (5, 0), u1 = e1, v1 = e3
    A = np.array([[0.0, 0.0, 5.0], [0.0, 0.0, 0.0]])
    V = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])   # columns e3, e1, e2
    assert O.paper_error(A, np.eye(2), np.array([5.0, 0.0]), V) == 0.0
    assert O.paper_error(A, np.eye(2), np.array([5.0, 0.0]), V.T) == pytest.approx(1.0)  # wrong V
    assert O.paper_error(A, np.eye(2), np.array([5.0, 0.0]), V, sigma_max=2.5) == 0.0


def test_column_residual_hand_cases():
    """column_residual (Q28): max_i ||A_hat v_i - sigma_i u_i||_2 / sigma_1, i < m."""
    A = np.array([[5.0, 0.3], [0.0, 1.4]])
    I = np.eye(2)
    # column 0 exact; column 1: (0.3, 1.4) - (0, 1) = (0.3, 0.4), 2-norm 0.5 (max-abs 0.4)
    assert O.column_residual(A, I, np.array([5.0, 1.0]), I) == pytest.approx(0.1, rel=1e-15)
    # A_hat^T instead of A_hat would give max(0.3, 0.4) / 5 = 0.08
    assert O.column_residual(A.T, I, np.array([5.0, 1.0]), I) == pytest.approx(0.08, rel=1e-15)
    # rectangular: only the m columns of V paired with U count
    A = np.array([[0.0, 0.0, 5.0], [0.0, 0.0, 0.0]])
    V = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    assert O.column_residual(A, np.eye(2), np.array([5.0, 0.0]), V) == 0.0
    V2 = V.copy()
    V2[:, 2] = 7.0  # the (n - m)-th column is not used
    assert O.column_residual(A, np.eye(2), np.array([5.0, 0.0]), V2) == 0.0
    # sigma_1 scales the result
    assert O.column_residual(A, np.eye(2), np.array([4.0, 0.0]), V) == pytest.approx(1.0 / 4.0)


def test_threaded_evaluation_is_bitwise_serial(monkeypatch):
    """The oracle evaluates independent roots on several threads; every root's sum is the
    same numpy reduction of the same row, so roots and w are bitwise the one-thread ones."""
    import oracle.svd1_oracle as M
    rng = np.random.default_rng(5)
    d, z, rho = random_secular(700, rng, kind="graded")
    monkeypatch.setattr(M, "THREADS", 1)
    k1, t1 = O.secular_roots_bisect(d, z, rho)
    w1 = O.secular_w(d, z, rho, k1, t1)
    monkeypatch.setattr(M, "THREADS", 7)
    k7, t7 = O.secular_roots_bisect(d, z, rho)
    w7 = O.secular_w(d, z, rho, k7, t7)
    assert np.array_equal(k1, k7) and np.array_equal(t1, t7) and np.array_equal(w1, w7)


# ------------------------------------------------------------- edge cases, reading D9
@pytest.mark.parametrize("name", EDGE_CASES)
def test_svd_update_edge_cases_vs_brute_force(name):
    """Degenerate inputs of Alg 6.1 (synth/edge.py: the smallest shapes, zero weights,
    rank-deficient and fully repeated spectra, extreme scales, unbalanced a b^T) against a
    brute-force one-sided Jacobi SVD of A_hat, with orthogonality and residual."""
    U, s, V, a, b = edge_case(name)
    m = U.shape[0]
    r = O.svd_update(U, s, V, a, b)
    A_hat = (U * s) @ V[:, :m].T + np.outer(a, b)
    f = math.ldexp(1.0, math.frexp(float(np.max(np.abs(A_hat))))[1])  # (exact rescaling: the
    _, sj, _ = jacobi_svd(A_hat / f)                                  #  brute force's own
    e = sigma_errors(r["sigma"], f * sj)                              #  thresholds are absolute)
    assert e["gram"] <= 1e-13 and e["rel_top"] <= 1e-12, e
    assert O.orth_defect(r["U"]) <= 1e-13 and O.orth_defect(r["V"]) <= 1e-13
    assert O.column_residual(A_hat, r["U"], r["sigma"], r["V"]) <= EDGE_RES_TOL.get(name, 1e-13)


@pytest.mark.parametrize("name", ["tiny33", "a_in_span", "rank_deficient", "scaled_down", "unbalanced"])
def test_balance_rescaling_bitwise(name):
    """Reading D9: (2^t a, b / 2^t) is the same rank-1 term; with the power-of-two balance
    factor the oracle returns bitwise the same factors for every t."""
    U, s, V, a, b = edge_case(name)
    r = O.svd_update(U, s, V, a, b)
    for t in (-30, -7, 5, 33):
        r2 = O.svd_update(U, s, V, a * 2.0 ** t, b / 2.0 ** t)
        for k in ("U", "sigma", "V"):
            assert np.array_equal(r[k], r2[k]), (name, t, k)


def test_balance_factor_cases():
    """balance_factor: c^2 within a factor of 4 of x / y, a power of two, 1 on degenerate norms."""
    for x, y in [(1.0, 1.0), (3.0, 1.0), (1e-30, 7.0), (5e200, 1e-100), (0.7, 0.3)]:
        c = O.balance_factor(x, y)
        assert math.frexp(c)[0] == 0.5 and 0.25 <= c * c / (x / y) <= 4.0, (x, y, c)
    assert O.balance_factor(0.0, 1.0) == 1.0 and O.balance_factor(1.0, 0.0) == 1.0
    assert O.balance_factor(float("inf"), 1.0) == 1.0


def test_unbalanced_needs_d9(monkeypatch):
    """Why D9: without the balance (c = 1) the paper's 2x2 Schur split cancels to
    eps ||a||^2 and the unbalanced and scaled-down cases lose all accuracy."""
    import oracle.svd1_oracle as OM
    monkeypatch.setattr(OM, "balance_factor", lambda x, y: 1.0)
    worst = 0.0
    for name in ("unbalanced", "scaled_down"):
        U, s, V, a, b = edge_case(name)
        m = U.shape[0]
        r = O.svd_update(U, s, V, a, b)
        A_hat = (U * s) @ V[:, :m].T + np.outer(a, b)
        worst = max(worst, O.column_residual(A_hat, r["U"], r["sigma"], r["V"]))
    assert worst > 1e-6
