"""Build libsvd1.so in-tree with nvcc for sm_100a (no torch types anywhere in the library)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
SOURCES = ["kernels_spectral.cu", "kernels_apply.cu", "svd1_host.cu"]
LIB = os.environ.get("SVD1_LIB_OUT") or os.path.join(HERE, "libsvd1.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


FLAGS += os.environ.get("SVD1_NVCC_EXTRA", "").split()  # e.g. -DSVD1_BOUNDS (debug checks)


def build(verbose=False, force=False):
    srcs = [os.path.join(SRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(SRC, "svd1_internal.cuh"),
                   os.path.join(os.path.dirname(HERE), "include", "svd1.h")]
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(p) <= t for p in deps):
            return LIB
    objs = []
    for s in srcs:
        o = os.path.join(SRC, os.path.basename(s) + ".o")
        cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {s}")
        objs.append(o)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
           "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
