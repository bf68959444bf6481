"""Time the CPU oracle (test infrastructure) on one C3 / C5 update with O8 sampled rows:
sizes the parity tests and the reference arm on the GPU box's host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from synth import config_inputs

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t0 = time.perf_counter()
inp = config_inputs(cfg, updates=1)
print("gen", time.perf_counter() - t0, flush=True)
U, s, V = inp["U"], inp["sigma"], inp["V"]
a, b = inp["ab"][0]
m, n = U.shape[0], V.shape[0]
rng = np.random.default_rng(99)
ru = np.sort(rng.choice(m, 96, replace=False)); rv = np.sort(rng.choice(n, 96, replace=False))
t0 = time.perf_counter()
d = s[::-1] ** 2
z = U.T @ a
k, tau = O.secular_roots_bisect(d, z[::-1], 1.0)
print("one bisection", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter()
O.loewner_zhat(d, k, tau, 1.0, z[::-1])
print("one loewner", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter()
O.svd_update(U, s, V, a, b, sign_rule="probe", rows=(ru, rv))
print("update O8", time.perf_counter() - t0, flush=True)
