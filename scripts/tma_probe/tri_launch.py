"""Diagnostic only: launch Triton's kernel (compiled by our ptxas) with our descriptor."""
import ctypes as C
import sys
import torch
torch.cuda.init()
a = torch.arange(100 * 152, dtype=torch.float64, device="cuda").reshape(100, 152)
out = torch.zeros(4096, dtype=torch.float64, device="cuda")
cu = C.CDLL("libcuda.so.1")
mine = (C.c_uint64 * 24)()
base = C.addressof(mine)
off = (64 - base % 64) % 64
mp = base + off
dims = (C.c_uint64 * 2)(152, 100)
strides = (C.c_uint64 * 1)(152 * 8)
box = (C.c_uint32 * 2)(16, 16)
es = (C.c_uint32 * 2)(1, 1)
print("enc", cu.cuTensorMapEncodeTiled(C.c_void_p(mp), 8, 2, C.c_void_p(a.data_ptr()), dims, strides, box, es, 0, 0, 1, 0))
mod = C.c_void_p()
print("load", cu.cuModuleLoad(C.byref(mod), sys.argv[1].encode()))
fn = C.c_void_p()
print("getfn", cu.cuModuleGetFunction(C.byref(fn), mod, b"k"))
cu.cuFuncSetAttribute(fn, 8, 9216)
p1, p2 = C.c_uint32(152), C.c_uint32(100)
p3, p4 = C.c_uint64(152), C.c_uint64(1)
po, p6, p7 = C.c_uint64(out.data_ptr()), C.c_uint64(0), C.c_uint64(0)
params = (C.c_void_p * 8)(mp, C.addressof(p1), C.addressof(p2), C.addressof(p3), C.addressof(p4), C.addressof(po),
                           C.addressof(p6), C.addressof(p7))
print("launch", cu.cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 8192 + 1024, C.c_void_p(torch.cuda.current_stream().cuda_stream), params, None))
try:
    torch.cuda.synchronize()
    print("OK", out[:3].tolist())
except Exception as e:
    print("FAIL", str(e)[:80])
