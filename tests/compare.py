"""Comparison helpers for parity tests (test-only; no method arithmetic).

Readings:
  D2   singular values: |s^2 - s*^2| <= 1e-12 s*_1^2 (Gram-normwise) and
       |s - s*| <= 1e-12 s*_i for s*_i >= 0.1 s*_1 (see sigma_errors).
  Q27  vectors: column i is compared up to sign when its relative eigengap
       min_j |s_i^2 - s_j^2| / s_1^2 >= gap_tol (default 1e-3); columns inside a
       cluster are compared through the orthogonal projector of the cluster.
"""
from __future__ import annotations

import numpy as np


def sigma_errors(s, s_ref):
    """Singular-value agreement (DESIGN.md §3.2 D2, reading of the north star's
    "relative error <= 1e-12"): the method computes sigma^2 as eigenvalues of the
    Gram matrices (STEP 8 P:350), whose rounding-level sensitivity is
    eps * sigma_1^2 in sigma^2.  Returns dict(gram = max|s^2 - s*^2| / s*_1^2,
    rel_top = max relative error over s*_i >= 0.1 s*_1, rel = max relative error
    over all s*_i > 0)."""
    s = np.asarray(s, np.float64)
    s_ref = np.asarray(s_ref, np.float64)
    s1 = float(np.max(np.abs(s_ref)))
    gram = float(np.max(np.abs(s * s - s_ref * s_ref)) / max(s1 * s1, 1e-300))
    rel = np.abs(s - s_ref) / np.maximum(s_ref, 1e-300)
    top = s_ref >= 0.1 * s1
    return dict(gram=gram, rel_top=float(np.max(rel[top])), rel=float(np.max(rel[s_ref > 0])) if np.any(s_ref > 0) else 0.0)


def clusters(eigs, gap_tol=1e-3):
    """Group indices (eigs sorted either way) whose consecutive relative gap
    |e_i - e_{i+1}| / max|e| < gap_tol."""
    e = np.asarray(eigs, np.float64)
    scale = max(float(np.max(np.abs(e))), 1e-300)
    groups, cur = [], [0]
    for i in range(1, e.size):
        if abs(e[i] - e[i - 1]) / scale < gap_tol:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def vector_error(Q, Q_ref, eigs_ref, gap_tol=1e-3, cols=None):
    """Max abs difference between column sets, up to sign for isolated columns,
    projector difference for clusters (Q27).  eigs_ref: eigenvalues (sigma^2 or
    D) in the column order of Q_ref.  cols limits the comparison to the first
    `cols` columns' clusters (clusters are taken whole)."""
    Q = np.asarray(Q, np.float64)
    Q_ref = np.asarray(Q_ref, np.float64)
    worst_iso, worst_clu, n_iso = 0.0, 0.0, 0
    for g in clusters(eigs_ref, gap_tol):
        if cols is not None and g[0] >= cols:
            continue
        if len(g) == 1:
            i = g[0]
            e = min(np.max(np.abs(Q[:, i] - Q_ref[:, i])), np.max(np.abs(Q[:, i] + Q_ref[:, i])))
            worst_iso = max(worst_iso, float(e))
            n_iso += 1
        else:
            A = Q[:, g]
            B = Q_ref[:, g]
            r = np.arange(0, A.shape[0], max(1, A.shape[0] // 1024))
            e = np.max(np.abs(A[r] @ A.T - B[r] @ B.T))
            worst_clu = max(worst_clu, float(e))
    return dict(isolated=worst_iso, cluster=worst_clu, n_isolated=n_iso)


def vector_error_rows(Qr, Qr_ref, eigs_ref, gap_tol=1e-3, cols=None):
    """vector_error on a row sample (rows are independent): isolated columns up to
    sign on the sampled entries; clusters through the projector restricted to the
    sampled rows, sum_c q_rc q_r'c."""
    return vector_error(Qr, Qr_ref, eigs_ref, gap_tol, cols)
