"""Comparison helpers for parity tests (test-only; no method arithmetic).

Readings:
  Q26  singular values: |s - s*| <= 1e-12 * s*_i for s*_i >= 1e-4 s*_1,
       else <= 1e-12 * s*_1.
  Q27  vectors: column i is compared up to sign when its relative eigengap
       min_j |s_i^2 - s_j^2| / s_1^2 >= gap_tol (default 1e-3); columns inside a
       cluster are compared through the orthogonal projector of the cluster.
"""
from __future__ import annotations

import numpy as np


def sigma_errors(s, s_ref):
    s = np.asarray(s, np.float64)
    s_ref = np.asarray(s_ref, np.float64)
    s1 = float(np.max(np.abs(s_ref)))
    big = s_ref >= 1e-4 * s1
    err = np.abs(s - s_ref)
    scale = np.where(big, s_ref, s1)
    return float(np.max(err / np.maximum(scale, 1e-300))), float(np.max(err / np.maximum(s_ref, 1e-300)))


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
            if A.shape[0] * A.shape[0] <= 16_000_000:
                e = np.max(np.abs(A @ A.T - B @ B.T))
            else:  # sampled-row projector entries
                r = np.arange(0, A.shape[0], max(1, A.shape[0] // 2048))
                e = np.max(np.abs(A[r] @ A.T - B[r] @ B.T))
            worst_clu = max(worst_clu, float(e))
    return dict(isolated=worst_iso, cluster=worst_clu, n_isolated=n_iso)
