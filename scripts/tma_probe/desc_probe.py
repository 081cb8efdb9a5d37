"""Diagnostic only: compare Triton's TMA descriptor with ours and launch our
probe kernel (probe2_arch.cubin, V1) with each, in one process."""
import ctypes as C
import sys

import torch
import triton  # noqa: F401
from triton.runtime import driver as tdrv

torch.cuda.init()
a = torch.arange(100 * 152, dtype=torch.float64, device="cuda").reshape(100, 152)
out = torch.zeros(4096, dtype=torch.float64, device="cuda")
utils = tdrv.active.utils

cu = C.CDLL("libcuda.so.1")
box_r, box_c = int(sys.argv[1]), int(sys.argv[2])
tdesc = utils.fill_tma_descriptor(a.data_ptr(), 0, 8, 8, [box_r, box_c], [100, 152], [152, 1], 0)
tbytes = C.string_at(id(tdesc) + 128, 128)

# our encoding (same call the product makes)
enc = cu.cuTensorMapEncodeTiled
mine = (C.c_uint64 * 16)()
dims = (C.c_uint64 * 2)(152, 100)
strides = (C.c_uint64 * 1)(152 * 8)
box = (C.c_uint32 * 2)(box_c, box_r)
es = (C.c_uint32 * 2)(1, 1)
rc = enc(C.byref(mine), 8, 2, C.c_void_p(a.data_ptr()), dims, strides, box, es, 0, 0, int(sys.argv[3]), 0)
mbytes = bytes(mine)
print("encode rc", rc)
for name, b in (("triton", tbytes), ("mine  ", mbytes)):
    w = [int.from_bytes(b[i * 8:i * 8 + 8], "little") for i in range(16)]
    print(name, " ".join(f"{x:016x}" for x in w[:8]))

mod = C.c_void_p()
print("load", cu.cuModuleLoad(C.byref(mod), b"scripts/tma_probe/probe2_arch.cubin"))
fn = C.c_void_p()
print("getfn", cu.cuModuleGetFunction(C.byref(fn), mod, b"_Z1kILi1EEv14CUtensorMap_stPKS0_Pdi"))
cu.cuFuncSetAttribute(fn, 8, 16 * 64 * 8 + 2048)  # MAX_DYNAMIC_SHARED_SIZE_BYTES
which = sys.argv[4]
buf = (C.c_uint64 * 24)()  # 64-B aligned storage for the map
addr = C.addressof(buf)
off = (64 - addr % 64) % 64
mapbuf = (C.c_char * 128).from_address(addr + off)
C.memmove(mapbuf, tbytes if which == "triton" else mbytes, 128)
gm = C.c_uint64(0)
op = C.c_uint64(out.data_ptr())
nb = C.c_int(box_r * box_c * 8)
params = (C.c_void_p * 4)(C.addressof(mapbuf), C.addressof(gm), C.addressof(op), C.addressof(nb))
stream = torch.cuda.current_stream().cuda_stream
r = cu.cuLaunchKernel(fn, 1, 1, 1, 128, 1, 1, 16 * 64 * 8 + 2048, C.c_void_p(stream), params, None)
print("launch", r)
try:
    torch.cuda.synchronize()
    print(which, "OK out0", out[0].item(), "expect", 5 * 152 + 3)
except Exception as e:
    print(which, "FAIL", str(e)[:100])
