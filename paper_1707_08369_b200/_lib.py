"""ctypes binding of libsvd1.so (include/svd1.h).  Argument marshalling only.

The library is loaded from this package directory (built in-tree by build.py);
there is no fallback: if the shared object is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsvd1.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsvd1.so not found at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (nvcc sm_100a) — there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

i64, i32, u32, dbl, vp = C.c_int64, C.c_int32, C.c_uint32, C.c_double, C.c_void_p
status_t = C.c_int


class Config(C.Structure):
    _fields_ = [("m", i64), ("n", i64), ("u_rows", i64), ("v_rows", i64), ("u_row0", i64),
                ("v_row0", i64), ("eps", dbl), ("stream", vp), ("flags", u32), ("fmm_min_n", i32),
                ("rank", i32), ("world", i32), ("nccl_id", vp)]


class Report(C.Structure):
    _fields_ = [("t_ms", dbl * 8), ("n_active", i32 * 4), ("n_deflated", i32 * 4),
                ("max_iter", i32 * 4), ("fmm_used", i32 * 4), ("p", i32), ("neg_clamped", i32),
                ("sign_flips", i32), ("noop", i32), ("kernel_launches", i64),
                ("apply_ms", dbl * 4), ("apply_flops", dbl * 4), ("spectral_ms", dbl * 4),
                ("fmm_levels", i32 * 4), ("fmm_max_near", i32 * 4), ("mean_iter", dbl * 4),
                ("pair_rotations", i32), ("apply_flops_exec", dbl * 4), ("gemm_ms", dbl * 4),
                ("allocations", i64), ("unpaired_clusters", i32)]

    def as_dict(self):
        return dict(t_ms=list(self.t_ms)[:7], n_active=list(self.n_active),
                    n_deflated=list(self.n_deflated), max_iter=list(self.max_iter),
                    fmm_used=list(self.fmm_used), p=self.p, neg_clamped=self.neg_clamped,
                    sign_flips=self.sign_flips, noop=self.noop,
                    kernel_launches=self.kernel_launches, apply_ms=list(self.apply_ms),
                    apply_flops=list(self.apply_flops), spectral_ms=list(self.spectral_ms),
                    fmm_levels=list(self.fmm_levels), fmm_max_near=list(self.fmm_max_near),
                    mean_iter=list(self.mean_iter), pair_rotations=self.pair_rotations,
                    apply_flops_exec=list(self.apply_flops_exec), gemm_ms=list(self.gemm_ms),
                    allocations=self.allocations, unpaired_clusters=self.unpaired_clusters)


def _sig(name, args):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = status_t
    return f


svd1_plan_create = _sig("svd1_plan_create", [C.POINTER(Config), C.POINTER(vp)])
svd1_plan_destroy = _sig("svd1_plan_destroy", [vp])
svd1_update = _sig("svd1_update", [vp, vp, i64, vp, vp, i64, vp, vp, dbl, C.POINTER(Report)])
svd1_update_batch = _sig("svd1_update_batch", [vp, vp, i64, vp, vp, i64, vp, i64, vp, i64, i64, dbl,
                                               C.POINTER(Report)])
svd1_update_batch_projected = _sig("svd1_update_batch_projected", [vp, vp, i64, vp, vp, i64, vp, vp, i64, i64,
                                                                   dbl, C.POINTER(Report)])
svd1_project = _sig("svd1_project", [vp, vp, i64, vp, i64, vp, vp, vp])
svd1_update_projected = _sig("svd1_update_projected",
                             [vp, vp, i64, vp, vp, i64, vp, vp, vp, dbl, C.POINTER(Report)])
svd1_cauchy_apply = _sig("svd1_cauchy_apply", [vp, i64, i64, vp, vp, vp, vp, vp, vp, i64, vp, i64,
                                               dbl, C.POINTER(i32)])
svd1_secular_solve = _sig("svd1_secular_solve", [vp, i64, vp, vp, dbl, vp, vp, C.POINTER(i32)])
svd1_loewner = _sig("svd1_loewner", [vp, i64, vp, vp, vp, dbl, vp, vp])
svd1_colnorms = _sig("svd1_colnorms", [vp, i64, vp, vp, vp, vp, vp])
svd1_fmm_tree_stats = _sig("svd1_fmm_tree_stats", [i64, vp, vp, vp, dbl, vp])
svd1_secfmm_plan_stats = _sig("svd1_secfmm_plan_stats", [i64, vp, vp])
svd1_nccl_unique_id = _sig("svd1_nccl_unique_id", [vp])
lib.svd1_status_string.argtypes = [status_t]
lib.svd1_status_string.restype = C.c_char_p
lib.svd1_version.argtypes = []
lib.svd1_version.restype = C.c_char_p

EXPORTS = ["svd1_plan_create", "svd1_plan_destroy", "svd1_update", "svd1_update_batch", "svd1_update_batch_projected", "svd1_project",
           "svd1_update_projected", "svd1_cauchy_apply", "svd1_secular_solve", "svd1_loewner",
           "svd1_colnorms", "svd1_fmm_tree_stats", "svd1_secfmm_plan_stats", "svd1_nccl_unique_id",
           "svd1_status_string", "svd1_version"]

FORCE_DIRECT = 0x1
FORCE_FMM = 0x2
SECULAR_FMM = 0x4     # secular solve with the FMM far field at every size > 64
SECULAR_DIRECT = 0x8  # secular solve with direct sums only
THIN_V = 0x10         # thin right factor: V is n x (m+1), column m workspace (svd1.h)
EMULATE_RANKS = 0x20  # world > 1 in one process: every rank's spectral slice computed here (tests)
FORCE_NCCL = 0x40     # NCCL all-gathers even at world 1 (tests the communicator path on one GPU)
FUSED_SIDE = 0x80     # fused per-side pass: X1 then X2 row chunk by row chunk


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for svd1_config.nccl_id (call on rank 0, broadcast to the others)."""
    buf = C.create_string_buffer(128)
    code = svd1_nccl_unique_id(C.cast(buf, vp))
    if code:
        raise RuntimeError(f"svd1_nccl_unique_id: {status_string(code)}")
    return buf.raw


def status_string(code: int) -> str:
    return lib.svd1_status_string(code).decode()


def version() -> str:
    return lib.svd1_version().decode()


def secfmm_plan_stats(d):
    """Host-only secular-FMM plan statistics (numpy ascending d): dict of svd1.h's 8 stats."""
    import numpy as np
    d = np.ascontiguousarray(d, dtype=np.float64)
    out = np.zeros(8, dtype=np.int64)
    code = svd1_secfmm_plan_stats(d.size, d.ctypes.data, out.ctypes.data)
    if code:
        raise RuntimeError(status_string(code))
    keys = ["L", "cells", "leaves", "m2l_parts", "near_ranges", "max_near_terms", "direct_roots", "plan_ns"]
    return dict(zip(keys, (int(x) for x in out)))


def fmm_tree_stats(d, k, tau, eps=1e-10):
    """Host-only FMM plan statistics (numpy inputs): dict of the 9 stats of svd1.h."""
    import numpy as np
    d = np.ascontiguousarray(d, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.int32)
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    out = np.zeros(9, dtype=np.int64)
    code = svd1_fmm_tree_stats(d.size, d.ctypes.data, k.ctypes.data, tau.ctypes.data, float(eps),
                               out.ctypes.data)
    if code:
        raise RuntimeError(status_string(code))
    keys = ["L", "cells", "max_leaf", "max_near", "near_pairs", "m2l_pairs", "flops_per_row", "tasks",
            "flops_exec_per_row"]
    return dict(zip(keys, (int(x) for x in out)))
