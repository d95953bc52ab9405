"""Build libsasbp.so in-tree with nvcc for sm_100a (no torch extension machinery: the library
is a plain C ABI, include/sasbp.h)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsasbp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sasbp.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build libsasbp.so (or an A/B variant at `out` with extra -D defines).  Every .cu is compiled
    to an object in parallel (the K2 instantiation families live in separate translation units),
    then linked."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    import concurrent.futures
    import tempfile
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
              "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines]]
    with tempfile.TemporaryDirectory(prefix="sasbp_build_") as tmpd:
        def one(src):
            obj = os.path.join(tmpd, os.path.basename(src) + ".o")
            subprocess.check_call(common + ["-c", "-o", obj, src])
            return obj
        srcs = sources()
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
            objs = list(ex.map(one, srcs))
        tmp = target + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    import sys
    args = [a for a in sys.argv[1:] if a != "-v"]
    out = None
    defs = []
    for a in args:
        if a.startswith("-D"):
            defs.append(a[2:])
        elif a.startswith("--out="):
            out = a[len("--out="):]
    print(build(force=True, verbose="-v" in sys.argv, out=out, defines=defs))
