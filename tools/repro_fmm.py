# Debug helper: run one standalone FMM Cauchy apply and report the error vs the oracle.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_1707_08369_b200 as P
from synth import interlaced_cauchy
n, rows, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda:0")
d, k, tau, zh, cs, uin = interlaced_cauchy(n, rows, seed)
want = O.cauchy_apply_explicit(uin, d, k, tau, zh, cs)
t = lambda x, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
plan = P.Plan(max(n, rows), max(n, rows), eps=1e-10, flags=P.FORCE_FMM)
out, used = plan.cauchy_apply(t(uin), t(d), t(k, torch.int32), t(tau), t(zh), t(cs))
torch.cuda.synchronize()
print("used", used, "err", float(np.max(np.abs(out.cpu().numpy() - want)) / np.max(np.abs(want))))
