"""Thin Python API over the C ABI (argument marshalling only: every step of the
path runs in libsvd1's CUDA kernels).  Tensors are torch CUDA float64, row-major;
int32 index arrays.  PyTorch supplies device memory and streams only."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L


class SVD1Error(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {L.status_string(code)} (status {code})")
        self.code = code


def _check(code, where):
    if code != 0:
        raise SVD1Error(code, where)


def _ptr(t, dtype=torch.float64, name="tensor"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() == 2:
        if t.stride(1) != 1:
            raise ValueError(f"{name} must be row-major (stride(1) == 1)")
    elif not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


def _ld(t):
    return t.stride(0)


class Plan:
    """svd1_plan: m x m U, n x n V (m <= n), eps -> Chebyshev order p.

    u_rows/v_rows/u_row0/v_row0 describe this process's row blocks (defaults:
    the whole matrices on one GPU)."""

    def __init__(self, m, n, eps=1e-10, stream=None, flags=0, fmm_min_n=0,
                 u_rows=None, v_rows=None, u_row0=0, v_row0=0, rank=0, world=1, nccl_id=None):
        """rank/world/nccl_id: one process per GPU (svd1.h); nccl_id = the 128 bytes of
        nccl_unique_id() from rank 0 (creation is then collective over the ranks)."""
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        self.m, self.n = int(m), int(n)
        self._id = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        cfg = L.Config(m=self.m, n=self.n, u_rows=self.m if u_rows is None else int(u_rows),
                       v_rows=self.n if v_rows is None else int(v_rows), u_row0=int(u_row0),
                       v_row0=int(v_row0), eps=float(eps),
                       stream=C.c_void_p(stream.cuda_stream), flags=int(flags),
                       fmm_min_n=int(fmm_min_n), rank=int(rank), world=int(world),
                       nccl_id=None if self._id is None else C.cast(self._id, C.c_void_p))
        self.cfg = cfg
        h = C.c_void_p()
        _check(L.svd1_plan_create(C.byref(cfg), C.byref(h)), "svd1_plan_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            L.svd1_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- Alg 6.1
    def update(self, U, sigma, V, a, b, eps=-1.0):
        """In-place rank-1 update: afterwards U diag(sigma) V[:, :m]^T = A + a b^T."""
        rep = L.Report()
        _check(L.svd1_update(self._h, _ptr(U, name="U"), _ld(U), _ptr(sigma, name="sigma"),
                             _ptr(V, name="V"), _ld(V), _ptr(a, name="a"), _ptr(b, name="b"),
                             float(eps), C.byref(rep)), "svd1_update")
        return rep.as_dict()

    def update_batch(self, U, sigma, V, A, B, eps=-1.0):
        """K in-place rank-1 updates in order: A (K x m), B (K x n) row-major, row t = a_t, b_t.
        Pipelined; returns the K reports."""
        K = A.shape[0]
        if A.dim() != 2 or B.dim() != 2 or B.shape[0] != K:
            raise ValueError("A, B must be K x m and K x n")
        reps = (L.Report * max(K, 1))()
        _check(L.svd1_update_batch(self._h, _ptr(U, name="U"), _ld(U), _ptr(sigma, name="sigma"),
                                   _ptr(V, name="V"), _ld(V), _ptr(A, name="A"), _ld(A),
                                   _ptr(B, name="B"), _ld(B), int(K), float(eps), reps),
               "svd1_update_batch")
        return [reps[t].as_dict() for t in range(K)]

    def update_batch_projected(self, U, sigma, V, projs, B=None, eps=-1.0):
        """Row-sharded stream after the projections: projs (K x proj_size) all-reduced;
        B (K x n, the full b's) only with THIN_V."""
        K = projs.shape[0]
        reps = (L.Report * max(K, 1))()
        _check(L.svd1_update_batch_projected(
            self._h, _ptr(U, name="U") if U is not None else None, _ld(U) if U is not None else 0,
            _ptr(sigma, name="sigma"), _ptr(V, name="V") if V is not None else None,
            _ld(V) if V is not None else 0, _ptr(projs, name="projs"),
            _ptr(B, name="B") if B is not None else None, _ld(B) if B is not None else 0,
            int(K), float(eps), reps),
            "svd1_update_batch_projected")
        return [reps[t].as_dict() for t in range(K)]

    def proj_size(self):
        return 5 * self.m + self.n + 6

    def project(self, U, V, a, b, proj):
        _check(L.svd1_project(self._h, _ptr(U, name="U") if U is not None else None,
                              _ld(U) if U is not None else 0,
                              _ptr(V, name="V") if V is not None else None,
                              _ld(V) if V is not None else 0, _ptr(a, name="a"),
                              _ptr(b, name="b"), _ptr(proj, name="proj")), "svd1_project")
        return proj

    def update_projected(self, U, sigma, V, proj, a, b, eps=-1.0):
        rep = L.Report()
        _check(L.svd1_update_projected(
            self._h, _ptr(U, name="U") if U is not None else None, _ld(U) if U is not None else 0,
            _ptr(sigma, name="sigma"), _ptr(V, name="V") if V is not None else None,
            _ld(V) if V is not None else 0, _ptr(proj, name="proj"), _ptr(a, name="a"),
            _ptr(b, name="b"), float(eps), C.byref(rep)), "svd1_update_projected")
        return rep.as_dict()

    # ------------------------------------------------------------- hooks
    def cauchy_apply(self, U_in, d, k, tau, zhat, colscale, U_out=None, eps=-1.0):
        rows, n = U_in.shape
        if U_out is None:
            U_out = torch.empty((rows, n), dtype=torch.float64, device=U_in.device)
        used = C.c_int32(0)
        _check(L.svd1_cauchy_apply(self._h, rows, n, _ptr(d, name="d"),
                                   _ptr(k, torch.int32, "k"), _ptr(tau, name="tau"),
                                   _ptr(zhat, name="zhat"), _ptr(colscale, name="colscale"),
                                   _ptr(U_in, name="U_in"), _ld(U_in), _ptr(U_out, name="U_out"),
                                   _ld(U_out), float(eps), C.byref(used)), "svd1_cauchy_apply")
        return U_out, bool(used.value)

    def secular_solve(self, d, z, rho):
        n = d.numel()
        k = torch.empty(n, dtype=torch.int32, device=d.device)
        tau = torch.empty(n, dtype=torch.float64, device=d.device)
        it = C.c_int32(0)
        _check(L.svd1_secular_solve(self._h, n, _ptr(d, name="d"), _ptr(z, name="z"), float(rho),
                                    _ptr(k, torch.int32, "k"), _ptr(tau, name="tau"),
                                    C.byref(it)), "svd1_secular_solve")
        return k, tau, it.value

    def loewner(self, d, k, tau, rho, z):
        zh = torch.empty_like(d)
        _check(L.svd1_loewner(self._h, d.numel(), _ptr(d, name="d"), _ptr(k, torch.int32, "k"),
                              _ptr(tau, name="tau"), float(rho), _ptr(z, name="z"),
                              _ptr(zh, name="zhat")), "svd1_loewner")
        return zh

    def colnorms(self, d, k, tau, zhat):
        out = torch.empty_like(d)
        _check(L.svd1_colnorms(self._h, d.numel(), _ptr(d, name="d"), _ptr(k, torch.int32, "k"),
                               _ptr(tau, name="tau"), _ptr(zhat, name="zhat"),
                               _ptr(out, name="colnorm")), "svd1_colnorms")
        return out


def update(U, sigma, V, a, b, eps=1e-10, **kw):
    """One-shot convenience: builds a plan and runs svd1_update in place."""
    plan = Plan(U.shape[0], V.shape[0], eps=eps, **kw)
    try:
        return plan.update(U, sigma, V, a, b)
    finally:
        plan.close()
