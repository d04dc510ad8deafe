"""In-tree build of libcavac_b200.so (sm_100a only) and of the C++ host
library libcavac_host.so (the reference-shaped cavac:: API over the C ABI).

    python -m paper_2112_00087_b200.build [--force]

Object files are cached under build/ keyed on source mtime; the shared
libraries land next to this file so they travel with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
CPP = os.path.join(PKG, "cpp")
BUILD = os.path.join(ROOT, "build", "cvk")
LIB = os.path.join(PKG, "libcavac_b200.so")
HOST_LIB = os.path.join(PKG, "libcavac_host.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include")]
CU_SOURCES = ["cvk_api.cu", "cvk_blas.cu", "cvk_krylov.cu", "cvk_phased.cu", "cvk_ddm.cu", "cvk_assemble.cu", "cvk_gmres.cu", "cvk_bicgl.cu", "cvk_rowblock.cu", "cvk_mmio.cu", "cvk_phased_g4.cu", "cvk_ilu.cu", "cvk_asm.cu"]
HEADERS = ["cvk_phased.cu", "cvk_complex.h", "cvk_engine.cuh", "cvk_kernels.h", "cvk_phased.h", "cvk_stream.cuh",
           "cvk_dcgs2.cuh", "cvk_tiles.cuh"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {os.path.basename(cmd[-1])}")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "cavac_b200.h")]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        if not os.path.exists(s):
            continue
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + NVFLAGS + ["-c", s, "-o", o])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(_run, jobs))
    if force or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl"])
    # C++ host API (namespace cavac) over the C ABI
    cpp_srcs = [os.path.join(CPP, f) for f in sorted(os.listdir(CPP))] if os.path.isdir(CPP) else []
    cpp_srcs = [f for f in cpp_srcs if f.endswith(".cpp")]
    if cpp_srcs:
        cpp_hdrs = [os.path.join(ROOT, "include", "cavac", f) for f in
                    os.listdir(os.path.join(ROOT, "include", "cavac"))] if os.path.isdir(
            os.path.join(ROOT, "include", "cavac")) else []
        if force or _stale(HOST_LIB, cpp_srcs + cpp_hdrs + [LIB]):
            _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                  "-I" + os.path.join(ROOT, "include"), "-o", HOST_LIB] + cpp_srcs +
                 ["-L" + PKG, "-lcavac_b200", "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
