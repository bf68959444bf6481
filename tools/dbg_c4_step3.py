import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1707_08369_b200 as P
dev = torch.device("cuda:0")
z = np.load("tools/c4_step3.npz")
d, zz, rho = z["d"], z["z"], float(z["rho"])
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.float64)
plan = P.Plan(8, 8)
k, tau, it = plan.secular_solve(T(d), T(zz), rho)
k, tau = k.cpu().numpy(), tau.cpu().numpy()
print("iters", it)
for j in (0, 1, len(d) - 1):
    print("j", j, "gpu k", k[j], "tau", repr(tau[j]), "mu", d[k[j]] + tau[j], "| oracle k", z["k"][j], "tau", repr(z["tau"][j]))
zh = plan.loewner(T(d), T(k.astype(np.int32)).to(torch.int32) if False else torch.from_numpy(k.astype(np.int32)).to(dev), T(tau), rho, T(zz)).cpu().numpy()
print("zhat finite", np.isfinite(zh).all(), zh[:3], "oracle", z["zhat"][:3])
cs = plan.colnorms(T(d), torch.from_numpy(k.astype(np.int32)).to(dev), T(tau), T(zh)).cpu().numpy()
print("colnorm finite", np.isfinite(cs).all(), cs[:3], "oracle 1/colnorm", 1 / z["colnorm"][:3])
