# torch.matmul fp64 8192^3 (cuBLAS DGEMM) as the practical FP64 ceiling; best of 10 and a ~3 s sustained loop.
import time, json, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); c = a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
t0 = time.time(); k = 0; e0.record()
while time.time() - t0 < 3.0:
    c = a @ b; k += 1
e1.record(); e1.synchronize(); sus = e0.elapsed_time(e1) / k
print(json.dumps({"mode": "torch_dgemm_8192", "burst_tflops": 2 * n**3 / best / 1e9, "sustained_tflops": 2 * n**3 / sus / 1e9}))
