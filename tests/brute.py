"""Brute-force reference routines used to PIN the oracle (test-only).

Textbook algorithms written out in full, independent of oracle/ and of the
CUDA path: cyclic Jacobi for symmetric eigenvalues, one-sided (Hestenes)
Jacobi SVD (the brute-force SVD named by BASELINE.json's north star and
SPEC.md:585).  Slow on purpose; use for n <= 64.
"""
from __future__ import annotations

import math

import numpy as np


def jacobi_eigvalsh(B, tol=1e-15, max_sweeps=60):
    """Cyclic Jacobi eigenvalue iteration on a symmetric matrix; ascending."""
    A = np.array(B, dtype=np.float64)
    n = A.shape[0]
    for _ in range(max_sweeps):
        off = math.sqrt(float(np.sum(np.triu(A, 1) ** 2)))
        if off <= tol * max(1e-300, math.sqrt(float(np.sum(A * A)))):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if apq == 0.0:
                    continue
                diff = A[q, q] - A[p, p]
                if abs(apq) < 1e-150 * abs(diff):
                    t = apq / diff
                else:
                    theta = diff / (2.0 * apq)
                    t = math.copysign(1.0, theta) / (abs(theta) + math.hypot(theta, 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                rp = A[p, :].copy()
                rq = A[q, :].copy()
                A[p, :] = c * rp - s * rq
                A[q, :] = s * rp + c * rq
                cp = A[:, p].copy()
                cq = A[:, q].copy()
                A[:, p] = c * cp - s * cq
                A[:, q] = s * cp + c * cq
    return np.sort(np.diag(A))


def jacobi_svd(A, tol=1e-15, max_sweeps=80):
    """One-sided Hestenes Jacobi SVD of A (m x n, m <= n).

    Orthogonalises the columns of W = A^T (n x m) by plane rotations applied on
    the right (accumulated in Q, m x m); at convergence W = V_m diag(s), so
    A = Q diag(s) V_m^T.  Returns (U = Q, s descending, V_m = W / s)."""
    W = np.array(A, dtype=np.float64).T.copy()
    n, m = W.shape
    Q = np.eye(m)
    for _ in range(max_sweeps):
        rotated = False
        for p in range(m - 1):
            for q in range(p + 1, m):
                alpha = float(W[:, p] @ W[:, p])
                beta = float(W[:, q] @ W[:, q])
                gamma = float(W[:, p] @ W[:, q])
                if abs(gamma) <= tol * math.sqrt(alpha * beta) or gamma == 0.0:
                    continue
                rotated = True
                zeta = (beta - alpha) / (2.0 * gamma)
                t = math.copysign(1.0, zeta) / (abs(zeta) + math.sqrt(1.0 + zeta * zeta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = c * t
                wp = W[:, p].copy()
                wq = W[:, q].copy()
                W[:, p] = c * wp - s * wq
                W[:, q] = s * wp + c * wq
                qp = Q[:, p].copy()
                qq = Q[:, q].copy()
                Q[:, p] = c * qp - s * qq
                Q[:, q] = s * qp + c * qq
        if not rotated:
            break
    s = np.sqrt(np.sum(W * W, axis=0))
    order = np.argsort(-s, kind="stable")
    s = s[order]
    Q = Q[:, order]
    W = W[:, order]
    Vm = W / np.where(s > 0, s, 1.0)[None, :]
    return Q, s, Vm
