"""Build libgear.so (the C-ABI of include/gear.h) for sm_100a, in-tree.

nvcc compiles every kernel with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3``; the host runtime is C++17.  NCCL comes from the torch-bundled
``nvidia/nccl`` wheel (rpath'd so the .so loads without LD_LIBRARY_PATH).
Objects are cached by mtime under ``paper_2310_05205_b200/build/``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# A/B variants (tools): GEAR_BUILD_VARIANT=name GEAR_NVCC_EXTRA="-DX=1" builds
# ab/libgear_<name>.so from build_<name>/ (load it with GEAR_LIB=...)
VARIANT = os.environ.get("GEAR_BUILD_VARIANT", "")
EXTRA = os.environ.get("GEAR_NVCC_EXTRA", "").split()
OBJ = os.path.join(HERE, "build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = (os.path.join(HERE, "ab", f"libgear_{VARIANT}.so") if VARIANT
       else os.path.join(HERE, "libgear.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    for base in [sysconfig.get_paths()["purelib"], *sys.path]:
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers (nvidia/nccl) not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def _headers() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "kernels", "*.cuh"))
            + [os.path.join(ROOT, "include", "gear.h")])


def build(force: bool = False, verbose: bool = False) -> str:
    nccl = _nccl_dir()
    os.makedirs(OBJ, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", *ARCH,
              "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"), *EXTRA]
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime)):
            continue
        cmd = [NVCC, *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed.append((src, out))
        elif verbose and out.strip():
            print(out)
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs,
                               "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                               "-Xlinker", "-rpath," + os.path.join(nccl, "lib")])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
