"""Diagnostics for one C3 update (GPU): host phase timing (SVD1_TIMING) and per-pass
FMM flops (SVD1_PASSSTATS) of the last update.  usage: python tools/diag_c3.py [cfg] [updates]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nup = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
inp = config_inputs(cfg_id, device=dev)
c = inp["cfg"]
U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
plan = P.Plan(c["m"], c["n"], eps=c["eps"])
for t in range(nup):
    if t == nup - 1:
        os.environ["SVD1_TIMING"] = "1"
        os.environ["SVD1_PASSSTATS"] = "1"
        print(f"--- update {t}", file=sys.stderr, flush=True)
    a, b = inp["ab"][t % len(inp["ab"])]
    rep = plan.update(U, s, V, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    torch.cuda.synchronize()
print({k: rep[k] for k in ("t_ms", "apply_ms", "apply_flops", "spectral_ms", "fmm_levels", "n_active")})

# realistic spectrum for host-side planning benchmarks: the first eigen-update of the
# next update (d = sigma^2 ascending, z = U^T a, rho ~ |b|^2), roots by the GPU solver
import numpy as np
a, b = inp["ab"][nup % len(inp["ab"])]
sg = s.cpu().numpy()
order = np.argsort(sg ** 2, kind="stable")
d = np.ascontiguousarray((sg ** 2)[order])
z = np.ascontiguousarray((U.T @ torch.from_numpy(a).to(dev)).cpu().numpy()[order])
rho = float(b @ b)
kk, tau, it = plan.secular_solve(torch.from_numpy(d).to(dev), torch.from_numpy(z).to(dev), rho)
kk, tau = kk.cpu().numpy(), tau.cpu().numpy()
if True:
    np.savez(os.path.join(ROOT, "gpurun_out", f"spectrum_c{cfg_id}.npz"), d=d, z=z, rho=rho, k=kk, tau=tau)
    print("saved spectrum", d.shape)

# per-pass device times of one update, sides serialized on one stream (diagnostics)
for env in ({"SVD1_NO_CHAIN": "1"}, {}):
    for k in ("SVD1_NO_CHAIN",):
        os.environ.pop(k, None)
    os.environ.update(env)
    os.environ["SVD1_ONE_STREAM"] = "1"
    os.environ["SVD1_PASSTIME"] = "1"
    os.environ.pop("SVD1_PASSSTATS", None)
    os.environ.pop("SVD1_TIMING", None)
    print("--- passtime", env, file=sys.stderr, flush=True)
    a, b = inp["ab"][nup % len(inp["ab"])]
    U2, s2, V2 = U.clone(), s.clone(), V.clone()
    rep = plan.update(U2, s2, V2, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    torch.cuda.synchronize()
    print("apply_ms", rep["apply_ms"], file=sys.stderr)
for k in ("SVD1_ONE_STREAM", "SVD1_PASSTIME", "SVD1_NO_CHAIN"):
    os.environ.pop(k, None)
