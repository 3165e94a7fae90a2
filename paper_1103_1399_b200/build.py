"""Build libqaa.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1103_1399_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libqaa.so")
SOURCES = ["api_context.cu", "api_tma.cu", "api_shard.cu", "api_evolve.cu", "api_observe.cu", "api_extras.cu", "kernels.cu", "pass_fast.cu", "pass_tma.cu", "spectrum.cu", "plan.cpp"]
HEADERS = ["api_internal.hpp", "kernels.cuh", "plan.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-Xptxas", "-v", "--expt-relaxed-constexpr", "-cudart", "static"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "qaa.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-Xlinker", "--no-undefined", "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        print(res.stdout + res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
