import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1707_08369_b200 as P
dev = torch.device("cuda:0")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.float64)
z = np.load("gpurun_out/c4fail_64.npz") if os.path.exists("gpurun_out/c4fail_64.npz") else np.load("tools/c4fail_64.npz")
for rep in range(3):
    U, s, V = T(z["U"]), T(z["s"]), T(z["V"])
    plan = P.Plan(U.shape[0], V.shape[0])
    r = plan.update(U, s, V, T(z["a"]), T(z["b"]))
    bad = (~torch.isfinite(V)).any(dim=0).nonzero().flatten().tolist()
    print("env one_stream=", os.environ.get("SVD1_ONE_STREAM"), "bad V cols", bad, "U finite", bool(torch.isfinite(U).all()), flush=True)
