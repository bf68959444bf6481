# Diagnostic: C5-recipe update at size n; per-column residuals and sign check.
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1707_08369_b200 as P
from synth import config_inputs
n = int(sys.argv[1]); flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda:0")
inp = config_inputs(5, device=dev, m=n, n=n, updates=1)
Ug, sg, Vg = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
a, b = (torch.from_numpy(x).to(dev) for x in inp["ab"][0])
A = (Ug * sg[None, :]) @ Vg.T + torch.outer(a, b)
plan = P.Plan(n, n, eps=1e-10, flags=flags)
rep = plan.update(Ug, sg, Vg, a, b)
R = A @ Vg - Ug * sg[None, :]
res = torch.linalg.norm(R, dim=0) / sg[0]
Rf = A @ (-Vg) - Ug * sg[None, :]
resf = torch.linalg.norm(Rf, dim=0) / sg[0]
bad = torch.nonzero(res > 1e-10).flatten().cpu().numpy()
print("n", n, "flags", flags, "max res", float(res.max()), "n bad", len(bad), "fixed by flip", int((resf[bad] < 1e-10).sum()) if len(bad) else 0)
print("rep", {k: rep[k] for k in ("n_active", "n_deflated", "sign_flips", "fmm_used", "max_iter")})
s = sg.cpu().numpy()
for i in bad[:10]:
    print(i, "sigma", s[i], "res", float(res[i]), "flipres", float(resf[i]), "neighbors", s[max(0,i-1):i+2])
