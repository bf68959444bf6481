"""Seeded generators (no method arithmetic here; see synth/__init__.py)."""
from __future__ import annotations

import math
import numpy as np

SEED_BASE = 170708369  # seed 170708369 + k for config Ck

# BASELINE.json "configs", in order C1..C5.
CONFIGS = {
    1: dict(name="C1", m=64, n=64, kind="gaussian", updates=1, ab_scale="1", eps=1e-10),
    2: dict(name="C2", m=1024, n=1024, kind="gaussian", updates=1, ab_scale="1/sqrt(n)", eps=1e-10),
    3: dict(name="C3", m=4096, n=4096, kind="graded", updates=16, ab_scale="1", eps=1e-10),
    4: dict(name="C4", m=2048, n=8192, kind="gaussian", updates=64, ab_scale="1e-2", eps=1e-10),
    5: dict(name="C5", m=16384, n=16384, kind="uniform_dup", updates=8, ab_scale="1", eps=1e-10),
}


def _rng(seed_or_rng):
    if isinstance(seed_or_rng, np.random.Generator):
        return seed_or_rng
    return np.random.default_rng(seed_or_rng)


def _qr_q(g, device):
    """Q factor of QR(g) with columns scaled by sign(diag R) (Haar measure)."""
    if device is None:
        q, r = np.linalg.qr(g)
        s = np.sign(np.diag(r))
        s[s == 0] = 1.0
        return np.ascontiguousarray(q * s[None, :])
    import torch
    t = torch.from_numpy(g).to(device)
    q, r = torch.linalg.qr(t)
    s = torch.sign(torch.diagonal(r))
    s[s == 0] = 1.0
    return (q * s[None, :]).contiguous()


def haar(n, seed_or_rng, device=None):
    """Random orthogonal n x n matrix; numpy array (device None) or torch tensor."""
    g = _rng(seed_or_rng).standard_normal((n, n))
    return _qr_q(g, device)


def gaussian_factors(m, n, seed_or_rng, device=None):
    """A with i.i.d. N(0,1) entries (m <= n) and its full SVD: U (m x m),
    sigma (m, descending), V (n x n) with A = U[:, :m] diag(sigma) V[:, :m]^T.
    The factorisation is LAPACK's (numpy) or torch.linalg.svd on `device`: input
    preparation, not the method under test."""
    rng = _rng(seed_or_rng)
    a = rng.standard_normal((m, n))
    if device is None:
        u, s, vt = np.linalg.svd(a, full_matrices=True)
        return np.ascontiguousarray(u), np.ascontiguousarray(s), np.ascontiguousarray(vt.T)
    import torch
    t = torch.from_numpy(a).to(device)
    u, s, vh = torch.linalg.svd(t, full_matrices=True)
    return u.contiguous(), s.contiguous(), vh.T.contiguous()


def graded_factors(n, seed_or_rng, device=None):
    """C3: A = Q1 diag(sigma) Q2^T, sigma_i = 10^(-6 i / n), i = 0..n-1
    (index base unstated in BASELINE.json; read as 0-based)."""
    rng = _rng(seed_or_rng)
    u = haar(n, rng, device)
    v = haar(n, rng, device)
    sig = 10.0 ** (-6.0 * np.arange(n) / n)
    if device is not None:
        import torch
        sig = torch.from_numpy(sig).to(device)
    return u, sig, v


def uniform_dup_sigma(n, rng, dup_frac=0.05):
    """C5 spectrum: sigma ~ U[1,100], with round(dup_frac*n) entries replaced by
    bitwise copies of uniformly chosen earlier entries; sorted descending."""
    n_dup = int(round(dup_frac * n))
    n_base = n - n_dup
    base = rng.uniform(1.0, 100.0, size=n_base)
    picks = rng.integers(0, n_base, size=n_dup)
    sig = np.concatenate([base, base[picks]])
    return np.sort(sig)[::-1].copy()


def uniform_dup_factors(n, seed_or_rng, device=None, dup_frac=0.05):
    rng = _rng(seed_or_rng)
    u = haar(n, rng, device)
    v = haar(n, rng, device)
    sig = uniform_dup_sigma(n, rng, dup_frac)
    if device is not None:
        import torch
        sig = torch.from_numpy(sig).to(device)
    return u, sig, v


def update_vectors(cfg_id, m, n, rng, count):
    """Rank-1 update vectors (a_k, b_k) per BASELINE.json configs."""
    out = []
    for _ in range(count):
        a = rng.standard_normal(m)
        b = rng.standard_normal(n)
        if cfg_id == 2:
            a /= math.sqrt(n)
            b /= math.sqrt(n)
        elif cfg_id == 4:
            a *= 1e-2
            b *= 1e-2
        out.append((a, b))
    return out


def config_inputs(cfg_id, device=None, m=None, n=None, updates=None):
    """Factors and update stream for config C<cfg_id>.  m, n, updates may be
    overridden to get the same recipe at a smaller size (parity-test cases)."""
    cfg = dict(CONFIGS[cfg_id])
    m = cfg["m"] if m is None else m
    n = cfg["n"] if n is None else n
    updates = cfg["updates"] if updates is None else updates
    rng = np.random.default_rng(SEED_BASE + cfg_id)
    if cfg["kind"] == "gaussian":
        u, s, v = gaussian_factors(m, n, rng, device)
    elif cfg["kind"] == "graded":
        assert m == n
        u, s, v = graded_factors(n, rng, device)
    else:
        assert m == n
        u, s, v = uniform_dup_factors(n, rng, device)
    ab = update_vectors(cfg_id, m, n, rng, updates)
    cfg.update(m=m, n=n, updates=updates)
    return dict(cfg=cfg, U=u, sigma=s, V=v, ab=ab)


def paper_uniform(m, n, seed_or_rng, lo=1.0, hi=9.0):
    """PAPER.md:411 (§7): "square and generated randomly with values ranging
    from [1,9]"; returns A (m x n), a (m), b (n) with entries U[lo, hi]."""
    rng = _rng(seed_or_rng)
    a_mat = rng.uniform(lo, hi, size=(m, n))
    a = rng.uniform(lo, hi, size=m)
    b = rng.uniform(lo, hi, size=n)
    return a_mat, a, b


def random_secular(n, seed_or_rng, rho=None, kind="gaussian", n_zero=0, n_dup=0):
    """A symmetric rank-one eigenproblem D + rho z z^T: d ascending, z, rho.
    kind: 'gaussian' d ~ N(0,1); 'graded' d = 10^(-12 i/n); 'uniform' d ~ U[1,100]^2;
    'wide' d = 10^(-140 .. 140) (products of a few gaps leave the double range).
    n_zero forced zero weights and n_dup bitwise-duplicated d values exercise
    deflation (SPEC.md:610 acceptance shape)."""
    rng = _rng(seed_or_rng)
    if kind == "gaussian":
        d = rng.standard_normal(n)
    elif kind == "graded":
        d = 10.0 ** (-12.0 * np.arange(n) / n)
    elif kind == "uniform":
        d = rng.uniform(1.0, 100.0, size=n) ** 2
    elif kind == "wide":
        d = 10.0 ** np.linspace(-140.0, 140.0, n)
    else:
        raise ValueError(kind)
    if n_dup:
        idx = rng.choice(n, size=n_dup, replace=False)
        src = rng.integers(0, n, size=n_dup)
        d[idx] = d[src]
    d = np.sort(d)
    z = rng.standard_normal(n)
    if n_zero:
        z[rng.choice(n, size=n_zero, replace=False)] = 0.0
    if rho is None:
        rho = float(rng.choice([-1.0, 1.0]) * rng.uniform(0.1, 10.0))
    return d, z, rho


def interlaced_cauchy(n, rows, seed_or_rng, rho_sign=1.0):
    """Sources d (ascending), roots in gap form (k, tau) strictly interlacing,
    weights zhat, column scales and a rows x n input block: inputs for the
    standalone Cauchy apply U_out = U_in diag(zhat) C diag(colscale),
    C_ij = 1/(d_i - mu_j) (Eq. CTildeFinalForm1)."""
    rng = _rng(seed_or_rng)
    d = np.sort(rng.standard_normal(n))
    gaps = np.diff(d)
    frac = rng.uniform(0.05, 0.95, size=n)
    k = np.arange(n, dtype=np.int32)
    tau = np.empty(n)
    if rho_sign > 0:
        tau[:-1] = frac[:-1] * gaps
        tau[-1] = frac[-1]
    else:
        tau[1:] = -frac[1:] * gaps
        tau[0] = -frac[0]
    zhat = rng.standard_normal(n)
    colscale = rng.uniform(0.5, 2.0, size=n)
    u_in = rng.standard_normal((rows, n))
    return d, k, tau, zhat, colscale, u_in
