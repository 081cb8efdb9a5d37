"""Diagnostic only: dump the SASS Triton generates around its TMA load."""
import torch
import triton
import triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor


@triton.jit
def k(desc, out_ptr):
    x = desc.load([0, 0])
    offs = tl.arange(0, 16)[:, None] * 64 + tl.arange(0, 64)[None, :]
    tl.store(out_ptr + offs, x)


a = torch.arange(100 * 152, dtype=torch.float64, device="cuda").reshape(100, 152)
desc = TensorDescriptor.from_tensor(a, [16, 64])
out = torch.empty(16 * 64, dtype=torch.float64, device="cuda")
kk = k.warmup(desc, out, grid=(1,))
open("gpurun_out/triton_k.cubin", "wb").write(kk.asm["cubin"])
open("gpurun_out/triton_full.ptx", "w").write(kk.asm["ptx"])
