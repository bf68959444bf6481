"""Timeline of a pipelined batch (svd1_update_batch) on the C3 workload: host stamps and
device events (SVD1_TIMELINE).  usage: python tools/diag_batch.py [K]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1707_08369_b200 as P
from synth import config_inputs

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dev = torch.device("cuda:0")
inp = config_inputs(3, device=dev)
U, s, V = inp["U"].clone(), inp["sigma"].clone(), inp["V"].clone()
A = torch.stack([torch.from_numpy(a) for a, _ in inp["ab"]]).to(dev)
B = torch.stack([torch.from_numpy(b) for _, b in inp["ab"]]).to(dev)
plan = P.Plan(4096, 4096, eps=1e-10)
plan.update_batch(U, s, V, A[:3], B[:3])
torch.cuda.synchronize()
os.environ["SVD1_TIMELINE"] = "1"
plan.update_batch(U, s, V, A[3:3 + K], B[3:3 + K])
torch.cuda.synchronize()
