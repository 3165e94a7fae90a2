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
SOURCES = ["api_context.cu", "api_tma.cu", "api_shard.cu", "api_evolve.cu", "api_observe.cu", "api_extras.cu", "kernels.cu", "pass_fast.cu", "pass_tma.cu", "pass_tmem.cu", "cluster_evolve.cu", "warp_evolve.cu", "spectrum.cu", "plan.cpp"]
HEADERS = ["api_internal.hpp", "kernels.cuh", "pass_common.cuh", "plan.hpp"]
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
    """Compile every translation unit in parallel (one nvcc per file), then link."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, cmd, r

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    link = [NVCC, *ARCH, "-cudart", "static", "-shared", "-Xlinker", "--no-undefined", "-o", LIB,
            *[o for o, _, _ in results], "-ldl"]
    lres = subprocess.run(link, capture_output=True, text=True) if all(r.returncode == 0 for _, _, r in results) \
        else None
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as f:
        for _, cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if lres is not None:
            f.write(" ".join(link) + "\n" + lres.stdout + lres.stderr)
    if lres is None or lres.returncode != 0:
        for _, _, r in results:
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
        if lres is not None:
            sys.stderr.write(lres.stdout + lres.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        print(open(log).read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
