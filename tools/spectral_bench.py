"""Spectral kernels (K2 secular, K3a Loewner, K3b norms) through the C-ABI test hooks at
C3 / C5 sizes, for ncu timing: python tools/spectral_bench.py [n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1707_08369_b200 as P
from synth import random_secular

dev = torch.device("cuda:0")
for n in [int(x) for x in sys.argv[1:]] or [4096, 16384]:
    rng = np.random.default_rng(n)
    d, z, rho = random_secular(n, rng, kind="uniform")
    plan = P.Plan(8, 8, eps=1e-10, flags=P.SECULAR_FMM if n >= 3072 else 0)
    T = lambda x, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
    dd, zz = T(d), T(z)
    for rep in range(3):
        k, tau, it = plan.secular_solve(dd, zz, rho)
        zh = plan.loewner(dd, k, tau, rho, zz)
        cn = plan.colnorms(dd, k, tau, zh)
    torch.cuda.synchronize()
    print(n, "ok", float(zh.abs().max()), float(cn.min()))
