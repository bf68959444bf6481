"""Plain, slow, fp64 numpy oracle of the paper's rank-1 SVD update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
PAPER.md line ("P:n") or SURVEY.md §8(c) reading ("Qn", "Rn", "On") it follows.
The oracle follows Algorithm 6.1 and Algorithm 6.2
step by step.  Library primitives used as single steps: numpy matmul (the
explicit products of P:337 and P:375, "explicit O(n^3) Cauchy product" of the
north star), numpy sum, sort, hypot, frexp.  No blocking, fusion or reordering
beyond what the paper states.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): closed forms and worked examples
(tests/golden/), brute-force one-sided Jacobi SVD / dense eigensolvers on tiny
inputs, invariants (interlacing, trace, orthogonality, residual, Frobenius and
Weyl identities).  Functions without such a pin would say "parity unpinned";
every function here has at least one (DESIGN.md §3.3 lists them).
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
import math
import os

import numpy as np

EPS = 2.0 ** -52  # fp64 unit roundoff x2 (machine epsilon)

_CHUNK_ELEMS = 1 << 22  # bound the n x n temporaries of the vectorised loops
# Independent roots are evaluated in parallel threads (numpy releases the GIL inside its
# loops).  Each root's sum is formed by the same numpy reduction over the same row
# whatever the chunking, so the results are bitwise those of one thread
# (tests/test_oracle_pins.py::test_threaded_evaluation_is_bitwise_serial).
THREADS = max(1, int(os.environ.get("SVD1_ORACLE_THREADS", os.cpu_count() or 1)))


# --------------------------------------------------------------------------- 2x2
def schur_sym_2x2(M):
    """Closed-form Schur (= eigen) decomposition of a symmetric 2x2 matrix.

    P:339-340 (Alg 6.1 STEPS 2-3, "Compute the Schur decomposition of"),
    P:538 (App. A).  Q31: for symmetric B the Schur form is the eigen-
    decomposition.  Returns (rho1, rho2, Q) with rho1 >= rho2, Q orthogonal and
    M = Q diag(rho1, rho2) Q^T.  The larger-magnitude eigenvalue comes from
    mean +/- radius and the other from det / big (no cancellation).
    """
    M = np.asarray(M, dtype=np.float64)
    p, q, r = M[0, 0], 0.5 * (M[0, 1] + M[1, 0]), M[1, 1]
    if not np.all(np.isfinite(M)):
        raise ValueError("NonFinite")
    if q == 0.0:
        if p >= r:
            return float(p), float(r), np.eye(2)
        return float(r), float(p), np.array([[0.0, 1.0], [1.0, 0.0]])
    mean = 0.5 * (p + r)
    rad = math.hypot(0.5 * (p - r), q)
    big = mean + math.copysign(rad, mean) if mean != 0.0 else rad
    small = (p * r - q * q) / big
    rho1, rho2 = (big, small) if big >= small else (small, big)
    # eigenvector of rho1 from the second row: q v0 + (r - rho1) v1 = 0
    v = np.array([rho1 - r, q])
    if abs(v[0]) + abs(v[1]) == 0.0:
        v = np.array([q, rho1 - p])
    v = v / math.hypot(v[0], v[1])
    Q = np.array([[v[0], -v[1]], [v[1], v[0]]])
    return float(rho1), float(rho2), Q


def schur_update_2x2(beta):
    """Schur split of [[beta, 1], [1, 0]] (Q4 order rho1 > 0 > rho2)."""
    return schur_sym_2x2(np.array([[beta, 1.0], [1.0, 0.0]]))


# --------------------------------------------------------------------- STEP 1
def prepare_update(U, sigma, V, a, b):
    """Alg 6.1 STEP 1, formed literally (O2):
    b~ = U Sigma V^T b, a~ = V Sigma^T U^T a, beta = b^T b, alpha = a^T a,
    D_u = Sigma Sigma^T (m), D_v = Sigma^T Sigma (n; n-m trailing zeros)."""
    m, n = U.shape[0], V.shape[0]
    sig = np.asarray(sigma, dtype=np.float64)
    Sigma = np.zeros((m, n))
    Sigma[np.arange(m), np.arange(m)] = sig
    b_tilde = U @ (Sigma @ (V.T @ b))
    a_tilde = V @ (Sigma.T @ (U.T @ a))
    Du = sig * sig
    Dv = np.concatenate([sig * sig, np.zeros(n - m)])
    return dict(b_tilde=b_tilde, a_tilde=a_tilde, beta=float(b @ b), alpha=float(a @ a),
                Du=Du, Dv=Dv)


# ------------------------------------------------------------------ deflation
@dataclass
class DeflationResult:
    """Output of the deflation rule (DESIGN.md §3.2 D1)."""
    d: np.ndarray            # eigenvalue per position after rotations
    z: np.ndarray            # weight per position after rotations (0 if deflated)
    active: np.ndarray       # positions that enter the secular equation (ascending)
    deflated: np.ndarray     # positions that pass through (eigenvalue d[i])
    ops: list = field(default_factory=list)  # ('house', idx, v)
    tol: float = 0.0


def _apply_ops_cols(ops, cols):
    """Apply the recorded Householder transforms to the columns of `cols`
    (in place): U_G <- U_G H, H = I - 2 v v^T / v^T v."""
    for _, idx, v in ops:
        blk = cols[:, idx]
        cols[:, idx] = blk - np.outer(blk @ v, v) * (2.0 / (v @ v))
    return cols


def _apply_ops_vec(ops, vec):
    """Same transforms on a coefficient vector: v' = H^T v = H v."""
    vec = vec.copy()
    for _, idx, v in ops:
        blk = vec[idx]
        vec[idx] = blk - v * ((blk @ v) * 2.0 / (v @ v))
    return vec


def deflate(d, z, rho):
    """Deflation of D + rho z z^T with d ascending (Bunch-Nielsen-
    Sorensen cases (1) "some values of a_bar ... are zero", (3) "eigenvalues with
    repetition"; case (2) "|a_bar| = 1" reads as z being a unit coordinate
    vector, which case (1) already covers).  The paper gives no tolerance; the
    reading (DESIGN.md §3.2 D1) deflates only what fp64 cannot represent:

      (i)   zero weight: deflate i if |z_i| <= 8 eps ||z||  (z_i is at the
            rounding level of the projection z = U^T a_1 that produced it);
      (iii) runs of bitwise-equal d among the survivors: one Householder
            H = I - 2 v v^T / v^T v maps z_run -> -sign(z_last) ||z_run|| e_last;
            all but the last member deflate with their (unchanged) eigenvalue.

    Nearly-equal but distinct d are NOT merged: the gap representation
    (Q6) separates any two distinct doubles, and merging them at an
    eps*||D + rho z z^T|| tolerance would cost the small singular values of
    graded spectra (C3) their relative accuracy (DESIGN.md §3.2 D1).
    """
    d = np.array(d, dtype=np.float64)
    z = np.array(z, dtype=np.float64)
    n = d.size
    if n == 0:
        return DeflationResult(d, z, np.zeros(0, np.int64), np.zeros(0, np.int64), [], 0.0)
    znorm = math.sqrt(float(z @ z))
    tol = 8.0 * EPS * znorm
    alive = np.ones(n, dtype=bool)
    ops = []
    # (i) zero components
    for i in range(n):
        if abs(z[i]) <= tol:
            alive[i] = False
            z[i] = 0.0
    # (iii) runs of bitwise-equal d among survivors
    surv = np.flatnonzero(alive)
    t = 0
    while t < surv.size:
        u = t
        while u + 1 < surv.size and d[surv[u + 1]] == d[surv[t]]:
            u += 1
        if u > t:
            idx = surv[t:u + 1].copy()
            zg = z[idx]
            nrm = math.sqrt(float(zg @ zg))
            alpha_h = -math.copysign(nrm, zg[-1])
            v = zg.copy()
            v[-1] -= alpha_h
            ops.append(("house", idx, v))
            z[idx] = 0.0
            z[idx[-1]] = alpha_h
            alive[idx[:-1]] = False
        t = u + 1
    active = np.flatnonzero(alive)
    deflated = np.flatnonzero(~alive)
    return DeflationResult(d, z, active, deflated, ops, tol)


# ----------------------------------------------------------- secular equation
def _chunks(n_rows, n_cols, parts=1):
    step = max(1, min(_CHUNK_ELEMS // max(1, n_cols), -(-n_rows // parts)))
    for s in range(0, n_rows, step):
        yield slice(s, min(n_rows, s + step))


def _for_chunks(fn, n_rows, n_cols):
    """fn(slice) for row chunks of an n_rows x n_cols evaluation, on THREADS threads."""
    chunks = list(_chunks(n_rows, n_cols, THREADS))
    if THREADS == 1 or len(chunks) == 1:
        for sl in chunks:
            fn(sl)
        return
    with ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(fn, chunks))


def secular_w(d, z, rho, k, tau):
    """w(mu) = 1 + rho sum_i z_i^2 / (d_i - mu) (P:107-109 Eq. GolubEigenvalUpdate,
    P:363 Alg 6.2 STEP 2) at mu_j = d_{k_j} + tau_j, evaluated in the gap form
    d_i - mu_j = (d_i - d_{k_j}) - tau_j (Q6 / S:149)."""
    d = np.asarray(d, np.float64)
    z2 = np.asarray(z, np.float64) ** 2
    k = np.asarray(k)
    tau = np.asarray(tau, np.float64)
    out = np.empty(tau.size)

    def chunk(sl):
        delta = (d[None, :] - d[k[sl]][:, None]) - tau[sl, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            out[sl] = 1.0 + rho * np.sum(z2[None, :] / delta, axis=1)
    _for_chunks(chunk, tau.size, d.size)
    return out


def _from_bits(b):
    return np.asarray(b, dtype=np.int64).view(np.float64)


def _to_bits(x):
    return np.asarray(x, dtype=np.float64).view(np.int64)


def secular_roots_bisect(d, z, rho):
    """All n roots of w by bisection on the IEEE bit pattern of |tau| (R3).

    d strictly ascending, z nonzero (deflated problem), rho != 0.  For rho < 0
    the reflected problem (-d reversed, z reversed, -rho) is solved and mapped
    back.  Root j < n-1 of a rho > 0 problem lies in (d_j, d_{j+1}) (interlacing,
    S:134): origin k_j = j if w(midpoint) >= 0 (tau in (0, gap/2]), else
    k_j = j+1 (tau in [-gap/2, 0)).  The last root lies in (d_{n-1}, d_{n-1} +
    rho ||z||^2] with origin n-1.  Bisection halves the integer bit pattern of
    |tau| until the bracket is two adjacent doubles, then returns the endpoint
    with the smaller |w|.  Returns (k int64, tau fp64), mu_j = d[k_j] + tau_j.
    """
    d = np.asarray(d, np.float64)
    z = np.asarray(z, np.float64)
    n = d.size
    if n == 0:
        return np.zeros(0, np.int64), np.zeros(0)
    if rho < 0:
        k, tau = secular_roots_bisect(-d[::-1], z[::-1], -rho)
        return (n - 1 - k)[::-1].copy(), (-tau)[::-1].copy()
    z2 = z * z
    k = np.empty(n, np.int64)
    sgn = np.ones(n)
    hi_val = np.empty(n)
    if n > 1:
        j = np.arange(n - 1)
        mid = (d[j + 1] - d[j]) / 2.0
        w_mid = secular_w(d, z, rho, j, mid)
        left = w_mid >= 0.0
        k[:-1] = np.where(left, j, j + 1)
        sgn[:-1] = np.where(left, 1.0, -1.0)
        hi_val[:-1] = mid
    k[-1] = n - 1
    sgn[-1] = 1.0
    hi_val[-1] = rho * float(np.sum(z2))
    lo = np.zeros(n, np.int64)
    hi = _to_bits(hi_val).copy()
    for _ in range(70):
        act = (hi - lo) > 1
        if not act.any():
            break
        mbits = lo + (hi - lo) // 2
        ia = np.flatnonzero(act)
        tm = sgn[ia] * _from_bits(mbits[ia])
        wm = secular_w(d, z, rho, k[ia], tm)
        go_lo = np.where(sgn[ia] > 0, wm < 0.0, wm >= 0.0)
        lo[ia] = np.where(go_lo, mbits[ia], lo[ia])
        hi[ia] = np.where(go_lo, hi[ia], mbits[ia])
    t_hi = sgn * _from_bits(hi)
    t_lo = sgn * _from_bits(lo)
    w_hi = np.abs(secular_w(d, z, rho, k, t_hi))
    w_lo = np.full(n, np.inf)
    ok = lo > 0
    if ok.any():
        w_lo[ok] = np.abs(secular_w(d, z, rho, k[ok], t_lo[ok]))
    tau = np.where(w_lo < w_hi, t_lo, t_hi)
    return k, tau


# -------------------------------------------------------------------- Loewner
def loewner_zhat(d, k, tau, rho, z):
    """Recompute z from the computed roots (Gu-Eisenstat / Loewner; north-star
    item (2), P:38 cites Gu et al.; R4):
        zhat_i^2 = |prod_j (mu_j - d_i)| / (|rho| prod_{j != i} |d_j - d_i|),
        mu_j - d_i = (d_{k_j} - d_i) + tau_j,  sign(zhat_i) = sign(z_i).
    Evaluated as a running product of ratios in index order j = 0..n-1 with
    frexp exponent rescaling after every factor (no logs)."""
    d = np.asarray(d, np.float64)
    n = d.size
    P = np.ones(n)
    E = np.zeros(n, np.int64)
    for j in range(n):
        num = (d[k[j]] - d) + tau[j]
        den = d[j] - d
        den[j] = 1.0
        P = P * (np.abs(num) / np.abs(den))
        P, e = np.frexp(P)
        E += e
    zhat2 = np.ldexp(P, E) / abs(rho)
    return np.sign(np.asarray(z, np.float64)) * np.sqrt(zhat2)


# ------------------------------------------------------------ Cauchy structure
def cauchy_X(d, k, tau, zhat):
    """C~ = diag(a_bar) C diag(||c_j||)^-1 with C_ij = 1/(lambda_i - mu_j)
    (P:194-208 Eq. CTildeFinalForm1; Alg 6.2 STEPS 3, 5, 7 P:365-377), using
    zhat for a_bar (R4) and the gap form for lambda_i - mu_j (Q6):
        X_ij = zhat_i / ((d_i - d_{k_j}) - tau_j),  ||c_j|| = (sum_i X_ij^2)^(1/2).
    Returns (X normalised, colnorm)."""
    d = np.asarray(d, np.float64)
    X = np.asarray(zhat, np.float64)[:, None] / ((d[:, None] - d[np.asarray(k)][None, :])
                                                 - np.asarray(tau, np.float64)[None, :])
    colnorm = np.sqrt(np.sum(X * X, axis=0))
    return X / colnorm[None, :], colnorm


def cauchy_apply_explicit(U_in, d, k, tau, zhat, colscale):
    """Explicit product U_out = U_in diag(zhat) C diag(colscale),
    C_ij = 1/((d_i - d_{k_j}) - tau_j): Alg 6.2 STEPS 4-7 with the
    product U_2 = U_1 C formed directly (the quantity FMM(lambda, mu, -U_1)
    approximates)."""
    d = np.asarray(d, np.float64)
    C = 1.0 / ((d[:, None] - d[np.asarray(k)][None, :]) - np.asarray(tau, np.float64)[None, :])
    U1 = np.asarray(U_in, np.float64) * np.asarray(zhat, np.float64)[None, :]  # STEP 4
    return (U1 @ C) * np.asarray(colscale, np.float64)[None, :]


# ----------------------------------------------------------- RankOneUpdate
def rank_one_update(U, D, rho, z=None, a1=None, carry=()):
    """Alg 6.2 RankOneUpdate(U, a1, D, rho), R1-R6.

    U: rows x n (columns = eigenvectors for D, any order; rows may be any row
    subset since rows are independent), D: n eigenvalues.  Either a1 (literal
    STEP 1 GEMV z = U^T a1, R1) or z (= U^T a1 supplied, O8 large mode) is given.
    carry: coefficient vectors v = U^T x, returned as U_new^T x (B7 chain).

    Steps: sort D ascending (stable) -> R1 -> R2 deflation -> R3 bisection ->
    R4 Loewner -> R5 X (STEPS 3, 5, 7) -> R6 explicit product U_active X
    (STEP 6) -> merge mu with the deflated eigenvalues (stable ascending,
    deflated first on ties, Q8).  Returns (U_new, D_new ascending, carry_new, info).
    """
    U = np.asarray(U, np.float64)
    D = np.asarray(D, np.float64)
    n = D.size
    perm = np.argsort(D, kind="stable")
    Us = U[:, perm].copy()
    Ds = D[perm].copy()
    if z is None:
        z = Us.T @ np.asarray(a1, np.float64)          # STEP 1
    else:
        z = np.asarray(z, np.float64)[perm]
    carry = [np.asarray(c, np.float64)[perm] for c in carry]
    info = dict(n=n)
    if rho == 0.0 or not np.any(z != 0.0):
        return Us, Ds, carry, dict(info, n_active=0, deflated=n)
    dfl = deflate(Ds, z, rho)                           # R2
    _apply_ops_cols(dfl.ops, Us)
    carry = [_apply_ops_vec(dfl.ops, c) for c in carry]
    act, dfx = dfl.active, dfl.deflated
    da, za = dfl.d[act], dfl.z[act]
    k, tau = secular_roots_bisect(da, za, rho)          # STEP 2, R3
    zhat = loewner_zhat(da, k, tau, rho, za)            # R4
    X, colnorm = cauchy_X(da, k, tau, zhat)             # STEPS 3, 5, 7
    U_act = Us[:, act] @ X                              # STEP 6 (explicit)
    mu = da[k] + tau
    # merge: stable ascending, deflated first on exact ties
    vals = np.concatenate([dfl.d[dfx], mu])
    flag = np.concatenate([np.zeros(dfx.size), np.ones(act.size)])
    pos = np.concatenate([dfx, np.arange(act.size)])
    order = np.lexsort((pos, flag, vals))
    cols = np.concatenate([Us[:, dfx], U_act], axis=1)[:, order]
    new_carry = []
    for c in carry:
        cn = np.concatenate([c[dfx], X.T @ c[act]])
        new_carry.append(cn[order])
    info.update(n_active=int(act.size), deflated=int(dfx.size), k=k, tau=tau, zhat=zhat,
                z=za, d_active=da, colnorm=colnorm, tol=dfl.tol, ops=len(dfl.ops))
    return cols, vals[order], new_carry, info


def sym_rank_one_eig(U, D, a1, rho):
    """Convenience: (U_new, D_new) of U D U^T + rho a1 a1^T via Alg 6.2."""
    Un, Dn, _, _ = rank_one_update(U, D, rho, a1=a1)
    return Un, Dn


# --------------------------------------------------------------- Alg 6.1
def balance_factor(x_norm, y_norm):
    """Reading D9: c = 2^floor(e / 2) where x_norm / y_norm = f 2^e,
    f in [0.5, 1) -- a power of two with c^2 within a factor of 4 of x_norm / y_norm (1 if
    either norm is 0 or not finite).  Alg 6.1 splits a side's symmetric update through the
    2x2 Schur form of [[beta, 1], [1, 0]], which is not invariant under the exact
    rewriting a b^T = (c a)(b / c)^T: with ||a|| >> ||A b|| the two eigen-updates
    rho1 a1 a1^T + rho2 b1 b1^T cancel to eps ||a||^2 (not eps ||a|| ||A b||).  Each side
    takes its own c so that its two vectors have comparable norms; a power of two keeps the
    rescaled vectors exact, and e (from the two norms' exponents) shifts by exactly 2t when
    the inputs are (2^t a, b / 2^t), so such inputs give bitwise the same result."""
    if not (x_norm > 0.0 and y_norm > 0.0 and math.isfinite(x_norm) and math.isfinite(y_norm)):
        return 1.0
    mx, ex = math.frexp(x_norm)
    my, ey = math.frexp(y_norm)
    _, e2 = math.frexp(mx / my)
    return math.ldexp(1.0, (ex - ey + e2) // 2)


def svd_update(U, sigma, V, a, b, sign_rule="explicit", probes=None, rows=None):
    """Alg 6.1 "Update SVD of rank-1 modified matrix using FMM",
    O1-O8, with the explicit product in place of the FMM.

    U (m x m), sigma (m, descending), V (n x n), m <= n (Q1); a (m), b (n).
    Returns dict(U, sigma, V, info): A + a b^T = U diag(sigma) V[:, :m]^T.

    sign_rule "explicit" (O7): flip v_i if u_i^T A_hat v_i < 0 with A_hat formed.
    sign_rule "probe" (O8 / Q11): 4 probes g_k, p_k = U_hat^T g_k and
    q_k = V_hat^T A_hat^T g_k carried through the small-vector chain;
    s_i = sign(q_{k*,i} p_{k*,i}), k* = argmax_k |p_{k,i}|.
    rows: optional (row_idx_U, row_idx_V) to materialise only those rows of the
    outputs (O8 large-n mode); the chained z and the spectral data stay exact.
    """
    U = np.asarray(U, np.float64)
    V = np.asarray(V, np.float64)
    sigma = np.asarray(sigma, np.float64)
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    m, n = U.shape[0], V.shape[0]
    if m > n or sigma.size != m or a.size != m or b.size != n:
        raise ValueError("DimensionMismatch")
    for x in (U, V, sigma, a, b):
        if not np.all(np.isfinite(x)):
            raise ValueError("NonFinite")
    if not np.any(a != 0.0) or not np.any(b != 0.0):     # O1: A_hat = A
        return dict(U=U.copy(), sigma=sigma.copy(), V=V.copy(), info=dict(noop=True))
    large = rows is not None
    # STEP 1, literal (O2)
    if not large:
        ing = prepare_update(U, sigma, V, a, b)
        b_tilde, a_tilde = ing["b_tilde"], ing["a_tilde"]
        alpha, beta = ing["alpha"], ing["beta"]
    else:
        alpha, beta = float(a @ a), float(b @ b)
    Du = sigma * sigma
    Dv = np.concatenate([Du, np.zeros(n - m)])
    xa = U.T @ a                       # U^T a
    yb = V.T @ b                       # V^T b
    # D9: per-side balance of the rank-1 term before the Schur split (exact rewriting):
    # U side [c_u a, b~ / c_u] with beta / c_u^2, V side [b / c_v, c_v a~] with alpha c_v^2
    if not large:
        c_u = balance_factor(float(np.linalg.norm(b_tilde)), math.sqrt(alpha))
        c_v = balance_factor(math.sqrt(beta), float(np.linalg.norm(a_tilde)))
    else:                              # ||b~|| = ||Sigma V^T b||, ||a~|| = ||Sigma^T U^T a|| (B7)
        c_u = balance_factor(float(np.linalg.norm(sigma * yb[:m])), math.sqrt(alpha))
        c_v = balance_factor(math.sqrt(beta), float(np.linalg.norm(sigma * xa)))
    # STEPS 2-3, Q2: right-side eigenvalues are rho3, rho4
    rho1, rho2, Qu = schur_update_2x2(beta / (c_u * c_u))
    rho3, rho4, Qv = schur_update_2x2(alpha * (c_v * c_v))
    if probes is None:
        probes = np.random.default_rng(12345).standard_normal((4, m))
    probes = np.asarray(probes, np.float64)
    carry_u, carry_v = [], []
    if sign_rule == "probe":
        xg = [U.T @ g for g in probes]
        carry_u = xg
        carry_v = [np.concatenate([sigma * x, np.zeros(n - m)]) + yb * float(a @ g)
                   for x, g in zip(xg, probes)]
    if not large:
        au, btu = c_u * a, b_tilde / c_u              # D9
        bv, atv = b / c_v, c_v * a_tilde
        a1 = Qu[0, 0] * au + Qu[1, 0] * btu          # [a b~] Q_u = [a1 b1]
        b1 = Qu[0, 1] * au + Qu[1, 1] * btu
        a2 = Qv[0, 0] * bv + Qv[1, 0] * atv          # [b a~] Q_v = [a2 b2]
        b2 = Qv[0, 1] * bv + Qv[1, 1] * atv
        # STEP 4, STEP 5 (Q3 reads "(U~, b1, D~, rho2)")
        Ut, Dt, cu, i1 = rank_one_update(U, Du, rho1, a1=a1, carry=carry_u)
        Uh, Dh, cu, i2 = rank_one_update(Ut, Dt, rho2, a1=b1, carry=cu)
        # STEP 6, STEP 7
        Vt, Dvt, cv, i3 = rank_one_update(V, Dv, rho3, a1=a2, carry=carry_v)
        Vh, Dvh, cv, i4 = rank_one_update(Vt, Dvt, rho4, a1=b2, carry=cv)
    else:
        ru, rv = rows
        sx = sigma * yb[:m] / c_u                     # U^T b~ = Sigma V^T b (B7), D9
        xu = c_u * xa
        z1 = Qu[0, 0] * xu + Qu[1, 0] * sx
        w1 = Qu[0, 1] * xu + Qu[1, 1] * sx
        sxa = c_v * np.concatenate([sigma * xa, np.zeros(n - m)])   # V^T a~ = Sigma^T U^T a
        ybv = yb / c_v
        z3 = Qv[0, 0] * ybv + Qv[1, 0] * sxa
        w3 = Qv[0, 1] * ybv + Qv[1, 1] * sxa
        Ut, Dt, cu, i1 = rank_one_update(U[ru], Du, rho1, z=z1, carry=[w1] + list(carry_u))
        Uh, Dh, cu, i2 = rank_one_update(Ut, Dt, rho2, z=cu[0], carry=cu[1:])
        Vt, Dvt, cv, i3 = rank_one_update(V[rv], Dv, rho3, z=z3, carry=[w3] + list(carry_v))
        Vh, Dvh, cv, i4 = rank_one_update(Vt, Dvt, rho4, z=cv[0], carry=cv[1:])
    # STEP 8: Sigma_n = sqrt(D_n), descending (O6); clamp negatives (Q13)
    Uh, Dh = Uh[:, ::-1], Dh[::-1]
    Vh, Dvh = Vh[:, ::-1], Dvh[::-1]
    neg = int(np.sum(Dh < 0))
    sig_hat = np.sqrt(np.maximum(Dh, 0.0))
    # O7 / Q11 pairing of V_hat with U_hat (D5): for each cluster of
    # numerically equal final eigenvalues (consecutive gap <= 64 eps D_1; singletons
    # are clusters of one), M = U_c^T A_hat V_c = sigma W with W orthogonal; W is
    # orthonormalised (QR, positive diagonal) and V_c <- V_c W^T.  For a singleton
    # this is the sign flip of u^T A_hat v < 0.
    flips, rotations = 0, 0
    tolc = 64 * EPS * max(Dh[0], 0.0)
    clusters, i0 = [], 0
    while i0 < m:
        i1 = i0 + 1
        while i1 < m and Dh[i1 - 1] - Dh[i1] <= tolc:
            i1 += 1
        clusters.append((i0, i1))
        i0 = i1
    if sign_rule == "explicit" and not large:
        A_hat = (U * sigma[None, :]) @ V[:, :m].T + np.outer(a, b)
        for (i0, i1) in clusters:
            if sig_hat[i0] <= 0:
                continue
            if i1 - i0 == 1:
                if Uh[:, i0] @ (A_hat @ Vh[:, i0]) < 0:
                    Vh[:, i0] = -Vh[:, i0]
                    flips += 1
                continue
            M = Uh[:, i0:i1].T @ (A_hat @ Vh[:, i0:i1])
            q, r = np.linalg.qr(M / sig_hat[i0])
            W = q * np.sign(np.diag(r))[None, :]
            Vh[:, i0:i1] = Vh[:, i0:i1] @ W.T
            rotations += 1
    elif sign_rule == "probe":
        P = np.stack([c[::-1] for c in cu])[:, :m]     # p_k in U_hat column order
        Qp = np.stack([c[::-1] for c in cv])[:, :m]    # q_k in V_hat column order
        kstar = np.argmax(np.abs(P), axis=0)
        cols = np.arange(m)
        s = np.sign(Qp[kstar, cols] * P[kstar, cols])
        s[s == 0] = 1.0
        for (i0, i1) in clusters:
            k = i1 - i0
            if k == 1 or k > P.shape[0] or sig_hat[i0] <= 0:
                continue
            Pc, Qc = P[:, i0:i1].T, Qp[:, i0:i1].T        # k x K:  Q_c = M^T P_c
            Mt = Qc @ Pc.T @ np.linalg.inv(Pc @ Pc.T)
            q, r = np.linalg.qr(Mt.T / sig_hat[i0])
            W = q * np.sign(np.diag(r))[None, :]
            Vh[:, i0:i1] = Vh[:, i0:i1] @ W.T
            s[i0:i1] = 1.0
            rotations += 1
        Vh[:, :m] = Vh[:, :m] * s[None, :]
        flips = int(np.sum(s < 0))
    info = dict(rho=(rho1, rho2, rho3, rho4), Qu=Qu, Qv=Qv, alpha=alpha, beta=beta,
                neg_clamped=neg, flips=flips, rotations=rotations, Dv_hat=Dvh, D_hat=Dh,
                updates=(i1, i2, i3, i4))
    return dict(U=Uh, sigma=sig_hat, V=Vh, info=info)


# ------------------------------------------------------------------ metrics
def paper_error(A_hat, U, sigma, V, sigma_max=None):
    """Error = max |(A_hat - U Sigma V^T) / max sigma_hat| (Eq. error);
    max sigma_hat of A_hat computed directly (Q24: largest singular value)."""
    m = U.shape[0]
    R = A_hat - (U * sigma[None, :]) @ V[:, :m].T
    if sigma_max is None:
        sigma_max = float(np.linalg.norm(A_hat, 2))
    return float(np.max(np.abs(R)) / sigma_max)


def orth_defect(M):
    """max |M^T M - I| (Q29)."""
    M = np.asarray(M, np.float64)
    return float(np.max(np.abs(M.T @ M - np.eye(M.shape[1]))))


def column_residual(A_hat, U, sigma, V):
    """max_i ||A_hat v_i - sigma_i u_i||_2 / sigma_1 over i < m (Q28)."""
    m = U.shape[0]
    R = A_hat @ V[:, :m] - U * sigma[None, :]
    return float(np.max(np.linalg.norm(R, axis=0)) / max(float(sigma[0]), 1e-300))
