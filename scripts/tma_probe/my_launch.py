"""Diagnostic only: launch kernel 'mk(map, gm, out, nbytes)' from a cubin with our descriptor."""
import ctypes as C
import sys
import torch
torch.cuda.init()
a = torch.arange(100 * 152, dtype=torch.float64, device="cuda").reshape(100, 152)
out = torch.zeros(4096, dtype=torch.float64, device="cuda")
cu = C.CDLL("libcuda.so.1")
buf = (C.c_uint64 * 24)()
mp = C.addressof(buf) + (64 - C.addressof(buf) % 64) % 64
dims = (C.c_uint64 * 2)(152, 100)
strides = (C.c_uint64 * 1)(152 * 8)
box = (C.c_uint32 * 2)(int(sys.argv[2]), int(sys.argv[3]))
es = (C.c_uint32 * 2)(1, 1)
assert cu.cuTensorMapEncodeTiled(C.c_void_p(mp), 8, 2, C.c_void_p(a.data_ptr()), dims, strides, box, es, 0, 0, 1, 0) == 0
mod = C.c_void_p()
assert cu.cuModuleLoad(C.byref(mod), sys.argv[1].encode()) == 0
fn = C.c_void_p()
assert cu.cuModuleGetFunction(C.byref(fn), mod, b"mk") == 0
cu.cuFuncSetAttribute(fn, 8, 16 * 64 * 8 + 2048)
gm, po, nb = C.c_uint64(0), C.c_uint64(out.data_ptr()), C.c_int(int(sys.argv[2]) * int(sys.argv[3]) * 8)
params = (C.c_void_p * 4)(mp, C.addressof(gm), C.addressof(po), C.addressof(nb))
assert cu.cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 16 * 64 * 8 + 2048, C.c_void_p(torch.cuda.current_stream().cuda_stream), params, None) == 0
try:
    torch.cuda.synchronize()
    print(sys.argv[1], "OK", out[:2].tolist(), "expect", [763.0, 764.0])
except Exception as e:
    print(sys.argv[1], "FAIL", str(e).splitlines()[0])
