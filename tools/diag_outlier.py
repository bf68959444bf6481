"""Catch the occasional slow C3 stream: 30 runs of the 20-update stream (svd1_update_batch),
per-run rate; for runs slower than 0.85 x the median, the per-update host times (t_ms[1]
spectral rounds, t_ms[2] apply planning, t_ms[4] total) and apply windows (t_ms[5])."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

dev = torch.device("cuda:0")
inp = config_inputs(3, device=dev)
ab = [(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)) for a, b in inp["ab"]]
K = 20
A = torch.stack([ab[t % 16][0] for t in range(K)]); B = torch.stack([ab[t % 16][1] for t in range(K)])
U0, s0, V0 = inp["U"], inp["sigma"], inp["V"]
st = torch.cuda.current_stream()
plan = P.Plan(4096, 4096, stream=st)
U, s, V = U0.clone(), s0.clone(), V0.clone()
runs = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    U.copy_(U0); s.copy_(s0); V.copy_(V0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(st)
    reps = plan.update_batch(U, s, V, A, B)
    e1.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    runs.append((K / (e0.elapsed_time(e1) / 1e3), wall, reps))
med = statistics.median(r[0] for r in runs)
print("rates", [round(r[0]) for r in runs])
for i, (rate, wall, reps) in enumerate(runs):
    if rate < float(os.environ.get("SLOW", "0.85")) * med:
        print(f"slow run {i}: {rate:.0f}/s wall {wall*1e3:.1f} ms")
        for t, r in enumerate(reps):
            print(f"  u{t}: host spectral {r['t_ms'][1]:.2f} plan {r['t_ms'][2]:.2f} total {r['t_ms'][4]:.2f} window {r['t_ms'][5]:.2f} L {r['fmm_levels']}")
fast = runs[[r[0] for r in runs].index(max(r[0] for r in runs))][2]
print("fastest run per update:")
for t, r in enumerate(fast):
    print(f"  u{t}: host spectral {r['t_ms'][1]:.2f} plan {r['t_ms'][2]:.2f} total {r['t_ms'][4]:.2f} window {r['t_ms'][5]:.2f} L {r['fmm_levels']} GF {[round(f/1e9,2) for f in r['apply_flops']]}")
