"""Diagnostics (GPU): two standalone FMM Cauchy applies on two streams at once vs alone."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1707_08369_b200 as P
from synth import interlaced_cauchy
dev = torch.device("cuda:0")
n, rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, int(sys.argv[2]) if len(sys.argv) > 2 else 8192
def mk(seed):
    d, k, tau, zh, cs, uin = interlaced_cauchy(n, rows, seed)
    t = lambda x, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
    return t(uin), t(d), t(k, torch.int32), t(tau), t(zh), t(cs)
A, B = mk(1), mk(2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
p1 = P.Plan(max(n, rows), max(n, rows), eps=1e-10, flags=P.FORCE_FMM, stream=s1)
p2 = P.Plan(max(n, rows), max(n, rows), eps=1e-10, flags=P.FORCE_FMM, stream=s2)
ref1, _ = p1.cauchy_apply(*A); torch.cuda.synchronize()
ref2, _ = p2.cauchy_apply(*B); torch.cuda.synchronize()
ref1, ref2 = ref1.clone(), ref2.clone()
for it in range(5):
    o1 = torch.empty_like(ref1); o2 = torch.empty_like(ref2)
    p1.cauchy_apply(*A, U_out=o1)
    p2.cauchy_apply(*B, U_out=o2)
    torch.cuda.synchronize()
    print(it, "diff1", float((o1 - ref1).abs().max()), "diff2", float((o2 - ref2).abs().max()), flush=True)
