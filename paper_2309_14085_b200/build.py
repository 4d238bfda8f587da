"""In-tree build of the native libraries (sm_100a).

    python -m paper_2309_14085_b200.build

produces ``paper_2309_14085_b200/lib/libh2g.so`` (CUDA matvec, include/h2g.h)
and ``libh2b.so`` (native C++/OpenMP operator builder, include/h2b.h).
The .so files are git-ignored but travel to the GPU box with the snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]

TARGETS = {
    "libh2g.so": (["h2g_plan.cu", "h2g_p2p_launch.cu"],
                  ["h2g_kernels.cuh", "h2g_stream.cuh", "h2g_p2p.cuh", "h2g_eval.cuh",
                   "h2g_p2p_batched.cuh", "h2g_mma_direct.cuh"], "h2g.h"),
    "libh2b.so": (["h2b_build.cpp"], [], "h2b.h"),
}
CXX = os.environ.get("H2_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
# no -march=native / -ffast-math: keep IEEE fp64 operation order (no FMA
# contraction) like numpy's separate ufunc passes in the reference ACA
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-mavx2", "-mno-fma",
            "-I", os.path.join(ROOT, "include")]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = True) -> dict:
    os.makedirs(LIBDIR, exist_ok=True)
    built = {}
    for name, (srcs, deps, header) in TARGETS.items():
        out = os.path.join(LIBDIR, name)
        src_paths = [os.path.join(CSRC, s) for s in srcs]
        dep_paths = src_paths + [os.path.join(CSRC, s) for s in deps] + [
            os.path.join(ROOT, "include", header), __file__]
        if force or _stale(out, dep_paths):
            if srcs[0].endswith(".cu"):
                # one object per translation unit, compiled concurrently, then linked
                objs, procs = [], []
                for sp in src_paths:
                    obj = os.path.join(LIBDIR, os.path.basename(sp) + ".o")
                    cmd = [NVCC, *ARCH, *NVFLAGS, "-c", "-o", obj, sp]
                    if verbose:
                        print(" ".join(cmd), file=sys.stderr)
                    procs.append((cmd, subprocess.Popen(cmd)))
                    objs.append(obj)
                for cmd, pr in procs:
                    if pr.wait() != 0:
                        raise subprocess.CalledProcessError(pr.returncode, cmd)
                cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs]
            else:
                cmd = [CXX, *CXXFLAGS, "-shared", "-o", out, *src_paths]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True)
        built[name] = out
    return built


if __name__ == "__main__":
    build(force="--force" in sys.argv)
