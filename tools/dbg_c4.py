"""Debug: rectangular (C4 recipe) update streams, per-update finiteness of the factors."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1707_08369_b200 as P
from synth import config_inputs
dev = torch.device("cuda:0")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.float64)
for (m, n, K) in ((128, 512, 4), (64, 256, 5)):
    inp = config_inputs(4, m=m, n=n, updates=K)
    U, s, V = T(inp["U"]), T(inp["sigma"]), T(inp["V"])
    plan = P.Plan(m, n)
    for t, (a, b) in enumerate(inp["ab"]):
        Vp, Up, sp = V.clone(), U.clone(), s.clone()
        try:
            r = plan.update(U, s, V, T(a), T(b))
        except Exception as e:
            print(m, n, t, "ERR", e); break
        bad = (~torch.isfinite(V)).any(dim=0).nonzero().flatten().tolist()
        print(m, n, t, {k: r[k] for k in ("n_active", "n_deflated", "max_iter", "fmm_used", "pair_rotations", "sign_flips", "neg_clamped")},
              "bad V cols", bad[:10], len(bad), "s", float(s[-1]), flush=True)
        if bad:
            np.savez(f"gpurun_out/c4fail_{m}.npz", U=Up.cpu().numpy(), s=sp.cpu().numpy(), V=Vp.cpu().numpy(), a=a, b=b)
            # V columns before the update: norms of the null-space block
            print("prev V finite", bool(torch.isfinite(Vp).all()), "orth prev", float((Vp.T @ Vp - torch.eye(n, device=dev, dtype=torch.float64)).abs().max()))
            break
