"""Diagnostic only (not product code): TMA with a HOST-encoded descriptor through Triton."""
import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def k(desc, out_ptr, BM: tl.constexpr, BN: tl.constexpr):
    x = desc.load([0, 0])
    offs = tl.arange(0, BM)[:, None] * BN + tl.arange(0, BN)[None, :]
    tl.store(out_ptr + offs, x)

a = torch.arange(64 * 64, dtype=torch.float64, device="cuda").reshape(64, 64)
o = torch.empty(32 * 16, dtype=torch.float64, device="cuda")
d = TensorDescriptor.from_tensor(a, [32, 16])
ck = k[(1,)](d, o, 32, 16)
torch.cuda.synchronize()
print("triton host-desc tma ok", torch.equal(o.reshape(32, 16), a[:32, :16]))
import re
for line in ck.asm["ptx"].splitlines():
    if re.search(r"tensormap|cp\.async\.bulk|mbarrier|fence|elect|\.param", line):
        print(line.strip())
