"""Diagnostic only (not product code): does a TMA tensor-descriptor load work on this box?"""
import torch, triton, triton.language as tl

@triton.jit
def k(in_ptr, out_ptr, M, N, BM: tl.constexpr, BN: tl.constexpr):
    desc = tl.make_tensor_descriptor(in_ptr, shape=[M, N], strides=[N, 1], block_shape=[BM, BN])
    x = desc.load([0, 0])
    offs = tl.arange(0, BM)[:, None] * BN + tl.arange(0, BN)[None, :]
    tl.store(out_ptr + offs, x)

def alloc(size, align, stream):
    return torch.empty(size, dtype=torch.int8, device="cuda")
triton.set_allocator(alloc)
a = torch.arange(64 * 64, dtype=torch.float32, device="cuda").reshape(64, 64)
o = torch.empty(32 * 32, dtype=torch.float32, device="cuda")
k[(1,)](a, o, 64, 64, 32, 32)
torch.cuda.synchronize()
print("triton tma ok", torch.equal(o.reshape(32, 32), a[:32, :32]))
asm = k.cache if hasattr(k, "cache") else None
ck = k[(1,)](a, o, 64, 64, 32, 32)
ptx = ck.asm["ptx"]
import re
for line in ptx.splitlines():
    if re.search(r"tensormap|cp\.async\.bulk|mbarrier|fence|elect", line):
        print(line.strip())
