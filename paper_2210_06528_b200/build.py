"""In-tree build of libmfadd_b200.so (sm_100a) with plain nvcc.

    python -m paper_2210_06528_b200.build      # or: build()

The shared library lands next to this file so it travels to the GPU box with
the repo snapshot (it is git-ignored, not gpurun-ignored).  Rebuilds only when
a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmfadd_b200.so")
LIB_DEBUG = os.path.join(HERE, "libmfadd_b200_debug.so")  # -DMFB_DEBUG: device-side bounds checks
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    """The NCCL torch itself loads (site-packages/nvidia/nccl).  Linking the
    same library (by path + rpath) keeps one libnccl.so.2 per process whatever
    the import order; the system copy is older and would satisfy the SONAME
    first if this library were loaded before torch."""
    try:
        import nvidia.nccl as nn  # noqa: F401
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except Exception:
        return None
    return base if os.path.exists(os.path.join(base, "lib", "libnccl.so.2")) else None
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-O3"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(ROOT, "include", "mfadd_b200.h")]
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib, deps):
        return lib
    objdir = os.path.join(HERE, "_build_debug" if debug else "_build")
    extra = ["-DMFB_DEBUG"] if debug else []
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    headers = [d for d in deps if not d.endswith((".cu", ".cpp"))]
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src] + headers):  # per-object: only changed units recompile
            continue
        ncl = _nccl_dir()
        inc = ["-I", os.path.join(ncl, "include")] if ncl else []
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *inc, "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-Wno-deprecated-gpu-targets", *FLAGS, "-x", "c++", "-I", CSRC, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"--- nvcc failed on {src}\n{out.decode(errors='replace')}\n")
        elif verbose and out:
            sys.stderr.write(out.decode(errors="replace"))
    if failed:
        raise RuntimeError("libmfadd_b200 build failed")
    tmp = lib + ".tmp"
    ncl = _nccl_dir()
    nccl = ["-L", os.path.join(ncl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(ncl, "lib")] \
        if ncl else ["-lnccl"]
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", *nccl, "-lrt", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(link))
    subprocess.run(link, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
