"""One FMM Cauchy apply at C3 size (4096 rows x 4096 columns, interlaced synthetic
spectrum) through the C-ABI test hook, alone on the GPU: run with SVD1_PASSTIME=1 for the
per-pass times (stderr), prints the mean apply time over 10 calls (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1707_08369_b200 as P
from synth import interlaced_cauchy

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda:0")
d, k, tau, zh, cs, uin = interlaced_cauchy(n, n, 7)
plan = P.Plan(n, n, eps=1e-10, flags=P.FORCE_FMM)
t = lambda x, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
args = (t(uin), t(d), t(k, torch.int32), t(tau), t(zh), t(cs))
for _ in range(3):
    plan.cauchy_apply(*args)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    plan.cauchy_apply(*args)
e1.record()
torch.cuda.synchronize()
print(f"apply n={n}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per call (host planning included)")
