"""Secular solve timing, direct vs FMM far field, at BASELINE sizes (diagnostic)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1707_08369_b200 as P
from synth import random_secular


def cases(n):
    rng = np.random.default_rng(1)
    for kind, rho in (("gaussian", 3.0), ("graded", 4096.0), ("uniform", -2.0)):
        d, z, _ = random_secular(n, rng, kind=kind)
        yield kind, d, z, rho
    d = np.sort(np.concatenate([10.0 ** (-12 * np.arange(n - 16) / n), 1.7e7 * (1 + rng.random(16))]))
    yield "outliers", d, rng.standard_normal(n), 1.0


def main():
    for n in (4096, 8192):
        pd = P.Plan(n, n, eps=1e-10, flags=P.SECULAR_DIRECT)
        pf = P.Plan(n, n, eps=1e-10, flags=P.SECULAR_FMM)
        for name, d, z, rho in cases(n):
            dt, zt = torch.tensor(d, device="cuda"), torch.tensor(z, device="cuda")
            out = []
            for p in (pd, pf):
                ts = []
                for _ in range(7):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    k, tau, it = p.secular_solve(dt, zt, rho)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                mu = d[k.cpu().numpy()] + tau.cpu().numpy()
                out.append((float(np.median(ts[2:])), it, mu))
            rel = np.max(np.abs(out[0][2] - out[1][2]) / np.abs(out[0][2]))
            print(f"n={n:5d} {name:9s} direct {out[0][0]*1e3:7.1f} us it {out[0][1]:3d} | "
                  f"fmm {out[1][0]*1e3:7.1f} us it {out[1][1]:3d} | max rel mu diff {rel:.2e}", flush=True)
        pd.close()
        pf.close()


if __name__ == "__main__":
    main()
