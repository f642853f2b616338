"""In-tree build of librgbid_b200.so (sm_100a) — called by __graft_entry__.build().

Every .cu is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo
--fmad=false`` (no FMA contraction: the mask-deciding per-pixel arithmetic must
round exactly like the reference source reads).  The host-only synth.cpp is
compiled with g++ -ffp-contract=off.  Output: paper_1807_08271_b200/_lib/.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# RGBID_BUILD_DIR: build an instrumented / variant library elsewhere (tools/)
OUT = os.environ.get("RGBID_BUILD_DIR") or os.path.join(HERE, "_lib")
LIB = os.path.join(OUT, "librgbid_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
            "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"]
# extra nvcc flags for instrumented builds (e.g. -DRGBID_TDIST_TRACE, tools/tdist_phases.py)
CU_FLAGS += os.environ.get("RGBID_NVFLAGS", "").split()
CU_SRCS = ["align_kernels.cu", "fusion_kernels.cu", "map_kernels.cu", "runtime.cu", "frontend.cu"]
CPP_SRCS = ["synth.cpp"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "rgbid_b200.h"))
    procs, objs = [], []
    for src in CU_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT, "obj", src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, *CU_FLAGS, "-c", s, "-o", o]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                                text=True)))
    for src in CPP_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT, "obj", src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
                   "-I", "/usr/local/cuda/include", "-c", s, "-o", o]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                                text=True)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if verbose and out:
            sys.stdout.write(out)
        if p.returncode != 0:
            sys.stdout.write(out)
            failed.append(src)
    if failed:
        raise RuntimeError(f"compilation failed: {failed}")
    if force or procs or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        subprocess.run(cmd, check=True)
    import ctypes
    ctypes.CDLL(LIB)  # fail the build on unresolved symbols
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
