"""Diagnostics (GPU): one C5 update, FMM vs forced-direct plan; per-column residuals."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1707_08369_b200 as P
from synth import config_inputs
dev = torch.device("cuda:0")
nn = int(sys.argv[1]) if len(sys.argv) > 1 else None
only = sys.argv[2] if len(sys.argv) > 2 else "fmm,direct"
inp = config_inputs(5, device=dev, updates=1, m=nn, n=nn)
m = n = inp["U"].shape[0]
a, b = (torch.from_numpy(x).to(dev) for x in inp["ab"][0])
A = (inp["U"] * inp["sigma"][None, :]) @ inp["V"].T + torch.outer(a, b)
out = {}
for name, flags in (("fmm", 0), ("direct", P.FORCE_DIRECT)):
    if name not in only:
        continue
    Ug, sg, Vg = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
    rep = P.Plan(m, n, eps=1e-10, flags=flags).update(Ug, sg, Vg, a, b)
    torch.cuda.synchronize()
    colres = (torch.linalg.norm(A @ Vg - Ug * sg[None, :], dim=0) / sg[0]).cpu().numpy()
    ou = (Ug.T @ Ug - torch.eye(m, device=dev, dtype=torch.float64)).abs().max(dim=0).values.cpu().numpy()
    ov = (Vg.T @ Vg - torch.eye(n, device=dev, dtype=torch.float64)).abs().max(dim=0).values.cpu().numpy()
    print(name, "res", colres.max(), "orthU", ou.max(), "orthV", ov.max(), "levels", rep["fmm_levels"],
          "defl", rep["n_deflated"], "rot", rep["pair_rotations"])
    bad = np.nonzero(colres > 1e-10)[0]
    print("  bad res cols:", len(bad), bad[:20], "orthU bad:", np.nonzero(ou > 1e-10)[0][:20],
          "orthV bad:", np.nonzero(ov > 1e-10)[0][:20])
    out[name] = (Ug, sg, Vg)
if len(out) == 2:
    print("sigma diff fmm-direct", float((out["fmm"][1] - out["direct"][1]).abs().max()))
