"""Diagnostic only: does a TMA tensor-descriptor load work on this box via Triton?"""
import torch
import triton
import triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor


@triton.jit
def k(desc, out_ptr):
    x = desc.load([0, 0])
    offs = tl.arange(0, 16)[:, None] * 64 + tl.arange(0, 64)[None, :]
    tl.store(out_ptr + offs, x)


for dt in (torch.float32, torch.float64):
    a = torch.arange(100 * 152, dtype=dt, device="cuda").reshape(100, 152)
    desc = TensorDescriptor.from_tensor(a, [16, 64])
    out = torch.empty(16 * 64, dtype=dt, device="cuda")
    try:
        k[(1,)](desc, out)
        torch.cuda.synchronize()
        print(dt, "ok", out[:3].tolist(), "expect", a[0, :3].tolist())
        asm = k.cache[0] if hasattr(k, "cache") else None
    except Exception as e:
        print(dt, "FAIL", repr(e)[:200])
        break

kk = k.warmup(desc, out, grid=(1,))
ptx = kk.asm["ptx"]
for line in ptx.splitlines():
    if any(t in line for t in ("cp.async.bulk", "mbarrier", "tensormap", "fence", ".param", ".target", ".version", "prefetch")):
        print(line.strip()[:200])
