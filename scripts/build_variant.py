"""Build an in-tree A/B variant of the library: recompile the named units with
extra defines and link them with the default build's other objects.

    python scripts/build_variant.py pf3 stream_tma.cu -DMFB_RL_PF=3
-> paper_2210_06528_b200/libmfadd_b200_pf3.so (select with MFADD_LIB_VARIANT=pf3)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06528_b200 import build as B  # noqa: E402

name = sys.argv[1]
units = [a for a in sys.argv[2:] if not a.startswith("-")]
defs = [a for a in sys.argv[2:] if a.startswith("-")]
B.build()
objdir = os.path.join(B.HERE, "_build")
vdir = os.path.join(B.HERE, "_build_" + name)
os.makedirs(vdir, exist_ok=True)
ncl = B._nccl_dir()
inc = ["-I", os.path.join(ncl, "include")] if ncl else []
objs, procs = [], []
for src in B.sources():
    base = os.path.basename(src)
    if base in units:
        obj = os.path.join(vdir, base + ".o")
        procs.append(subprocess.Popen([B.NVCC, *B.ARCH, *B.FLAGS, *defs, *inc, "-I", B.CSRC, "-I",
                                       os.path.join(ROOT, "include"), "-c", src, "-o", obj]))
    else:
        obj = os.path.join(objdir, base + ".o")
    objs.append(obj)
for p in procs:
    if p.wait() != 0:
        raise SystemExit("variant build failed")
lib = os.path.join(B.HERE, f"libmfadd_b200_{name}.so")
nccl = ["-L", os.path.join(ncl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(ncl, "lib")] \
    if ncl else ["-lnccl"]
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", *nccl, "-lrt", "-ldl", "-lpthread"],
               check=True)
print(lib)
