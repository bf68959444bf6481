"""Per-update FMM plan statistics of the C3 stream through svd1_update_batch (20 updates, the
stream wrapping after 16 as bench.py's timed region does): tree depth, algorithmic flops
per apply, active sizes, per-update apply windows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

dev = torch.device("cuda:0")
inp = config_inputs(3, device=dev)
ab = [(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)) for a, b in inp["ab"]]
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
A = torch.stack([ab[t % 16][0] for t in range(K)]); B = torch.stack([ab[t % 16][1] for t in range(K)])
U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
plan = P.Plan(4096, 4096)
plan.update_batch(U.clone(), s.clone(), V.clone(), A, B)
reps = plan.update_batch(U, s, V, A, B)
for t, r in enumerate(reps):
    print(t, "L", r["fmm_levels"], "GF/apply", [round(f / 1e9, 2) for f in r["apply_flops"]], "near", r["fmm_max_near"],
          "win ms", round(r["t_ms"][5], 3), "top sigma", round(float(s[0]), 1) if t == K - 1 else "")
