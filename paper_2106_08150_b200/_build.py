"""Compile libmc.so (all CUDA sources, sm_100a) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libmc.so")
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh"))
                  + [os.path.join(ROOT, "include", "mc.h")])


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    srcs = sources()
    lib = out or LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(s) for s in srcs):
        return lib
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        nvcc = "nvcc"
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I" + os.path.join(ROOT, "include"),
           *[s for s in srcs if s.endswith(".cu")], "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(PKG, "csrc", "ptxas.log"), "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2:  # python -m paper_2106_08150_b200._build OUT.so DEF1 DEF2 ... (A/B variants)
        print(build(force=True, out=sys.argv[1], defines=sys.argv[2:]))
    else:
        print(build(force=True, verbose=True))
