"""Pipeline fill and drain of a 20-update C3 stream (svd1_update_batch, SVD1_TIMELINE):
the stream is warmed up on a copy, then the timed-like batch runs with device events; prints
update 0's and the last update's events.  usage: python tools/diag_fill.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

dev = torch.device("cuda:0")
inp = config_inputs(3, device=dev)
K = 20
A = torch.stack([torch.from_numpy(inp["ab"][t % 16][0]) for t in range(K)]).to(dev)
B = torch.stack([torch.from_numpy(inp["ab"][t % 16][1]) for t in range(K)]).to(dev)
plan = P.Plan(4096, 4096, eps=1e-10)
for _ in range(2):
    U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
    plan.update_batch(U, s, V, A, B)
torch.cuda.synchronize()
U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
torch.cuda.synchronize()
os.environ["SVD1_TIMELINE"] = "1"
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
plan.update_batch(U, s, V, A, B)
e1.record()
torch.cuda.synchronize()
print(f"stream: {e0.elapsed_time(e1):.3f} ms for {K} updates")
