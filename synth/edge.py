"""Seeded degenerate-case inputs for whole updates (no method arithmetic; see
synth/__init__.py): the edge cases of Alg 6.1 that the config recipes do not
reach -- the smallest shapes, update vectors inside a few singular directions (weights of
exact zero, S:128-129 deflation), rank-deficient and fully repeated spectra, extreme
scales of A and of the update, and unbalanced factors a b^T = (c a)(b / c)^T (reading D9).
edge_case(name) -> (U, sigma, V, a, b) with A = U diag(sigma) V[:, :m]^T, m <= n."""
from __future__ import annotations

import numpy as np

from .gen import haar

EDGE_CASES = ["tiny11", "tiny22", "tiny13", "tiny25", "tiny33", "a_in_span", "b_one_dir",
              "rank_deficient", "all_equal", "scaled_up", "scaled_down", "small_update",
              "large_update", "unbalanced", "downdate_top", "zero_matrix", "coordinate_update",
              "b_null_space"]
_TINY = {"tiny11": (1, 1), "tiny22": (2, 2), "tiny13": (1, 3), "tiny25": (2, 5), "tiny33": (3, 3)}
EDGE_SEED = 1000
# column residual bound per case where the method's own accuracy is looser than the north
# star's 1e-10: an exact zero singular value of A_hat comes out of the Gram eigenvalues
# as sqrt(O(eps) sigma_1^2), so reading D2's 1e-12 sigma_1^2 allows a residual
# of sqrt(1e-12) = 1e-6 on that column
EDGE_RES_TOL = {"downdate_top": 1e-6}


def edge_case(name, m=48):
    """The inputs of one edge case (seed EDGE_SEED + its index); m = n except tinyMN."""
    rng = np.random.default_rng(EDGE_SEED + EDGE_CASES.index(name))

    def fac(m_, n_, sig):
        return haar(m_, rng), np.asarray(sig, np.float64), haar(n_, rng)

    def spread(m_):
        return np.sort(rng.uniform(1.0, 10.0, m_))[::-1].copy()

    if name in _TINY:
        mm, nn = _TINY[name]
        U, s, V = fac(mm, nn, np.sort(rng.uniform(0.5, 2.0, mm))[::-1].copy())
        return U, s, V, rng.standard_normal(mm), rng.standard_normal(nn)
    n = m
    if name == "a_in_span":       # U^T a has two nonzeros: every other weight deflates
        U, s, V = fac(m, n, spread(m))
        return U, s, V, 2.0 * U[:, 0] + U[:, 3], rng.standard_normal(n)
    if name == "b_one_dir":       # V^T b = 3 e_5
        U, s, V = fac(m, n, spread(m))
        return U, s, V, rng.standard_normal(m), 3.0 * V[:, 5]
    if name == "rank_deficient":  # rank 5: sigma_5.. = 0 (a repeated zero eigenvalue)
        sig = np.zeros(m)
        sig[:5] = [5.0, 4.0, 3.0, 2.0, 1.0]
        U, s, V = fac(m, n, sig)
        return U, s, V, rng.standard_normal(m), rng.standard_normal(n)
    if name == "all_equal":       # A = 2 Q1 Q2^T: one eigenvalue of multiplicity m
        U, s, V = fac(m, n, np.full(m, 2.0))
        return U, s, V, rng.standard_normal(m), rng.standard_normal(n)
    if name in ("scaled_up", "scaled_down"):  # A and a b^T both scaled by 1e80 / 1e-20
        f = 1e80 if name == "scaled_up" else 1e-20
        U, s, V = fac(m, n, f * spread(m))
        return U, s, V, np.sqrt(f) * rng.standard_normal(m), np.sqrt(f) * rng.standard_normal(n)
    if name == "small_update":    # ||a b^T|| ~ 1e-11 ||A||
        U, s, V = fac(m, n, spread(m))
        return U, s, V, 1e-12 * rng.standard_normal(m), rng.standard_normal(n)
    if name == "large_update":    # ||a b^T|| ~ 1e9 ||A||
        U, s, V = fac(m, n, spread(m))
        return U, s, V, 1e6 * rng.standard_normal(m), 1e3 * rng.standard_normal(n)
    if name == "unbalanced":      # a b^T of unit size written as (1e8 a)(1e-8 b)^T
        U, s, V = fac(m, n, spread(m))
        return U, s, V, 1e8 * rng.standard_normal(m), 1e-8 * rng.standard_normal(n)
    if name == "downdate_top":    # a b^T = -sigma_1 u_1 v_1^T: A_hat has an exact zero singular value
        U, s, V = fac(m, n, spread(m))
        return U, s, V, -s[0] * U[:, 0], V[:, 0].copy()
    if name == "zero_matrix":     # A = 0: A_hat = a b^T, every other singular value 0
        U, s, V = fac(m, n, np.zeros(m))
        return U, s, V, rng.standard_normal(m), rng.standard_normal(n)
    if name == "coordinate_update":  # a = e_3, b = e_7 (one entry of A changes)
        U, s, V = fac(m, n, spread(m))
        a, b = np.zeros(m), np.zeros(n)
        a[3], b[7] = 1.0, 1.0
        return U, s, V, a, b
    if name == "b_null_space":    # m < n, b orthogonal to the row space of A (V^T b has no first m part)
        mm, nn = 24, 40
        U, s, V = fac(mm, nn, np.sort(rng.uniform(1.0, 10.0, mm))[::-1].copy())
        return U, s, V, rng.standard_normal(mm), V[:, mm:] @ rng.standard_normal(nn - mm)
    raise KeyError(name)
