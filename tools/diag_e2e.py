"""Run-to-run timing of the C3 stream through svd1_update_batch inside one process: value-style
(inputs resident) and e2e-style (a, b copied from pinned host memory each step), alternated,
after a per-update-API run, to locate the e2e leg's variance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

dev = torch.device("cuda:0")
inp = config_inputs(3, device=dev)
ab = [(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)) for a, b in inp["ab"]]
A = torch.stack([a for a, _ in ab]); B = torch.stack([b for _, b in ab])
A_h, B_h = A.cpu().pin_memory(), B.cpu().pin_memory()
U0, s0, V0 = inp["U"], inp["sigma"], inp["V"]
st = torch.cuda.current_stream()
plan = P.Plan(4096, 4096, stream=st)
U, s, V = U0.clone(), s0.clone(), V0.clone()
def restore():
    U.copy_(U0); s.copy_(s0); V.copy_(V0); torch.cuda.synchronize()
def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    restore(); e0.record(st); fn(); e1.record(st); torch.cuda.synchronize()
    return 16 / (e0.elapsed_time(e1) / 1e3)
def val():
    plan.update_batch(U, s, V, A, B)
def e2e():
    Ad, Bd = torch.empty_like(A), torch.empty_like(B)
    Ad.copy_(A_h, non_blocking=True); Bd.copy_(B_h, non_blocking=True)
    plan.update_batch(U, s, V, Ad, Bd)
for i in range(3):
    val()
restore()
for t in range(3):
    plan.update(U, s, V, A[t], B[t])
out = []
for i in range(6):
    out.append(("val", round(timed(val), 1)))
    out.append(("e2e", round(timed(e2e), 1)))
print(out)
restore()
for t in range(8):
    plan.update(U, s, V, A[t], B[t])
print("after per-update API:", round(timed(e2e), 1), round(timed(val), 1), round(timed(e2e), 1))
