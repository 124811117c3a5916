"""Build the in-tree C-ABI shared library libftk.so with nvcc for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, one object per source, linked with
-shared into paper_1905_12317_b200/libftk.so (git-ignored, shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libftk.so")
SOURCES = ["ftk_plan_math.cpp", "ftk_nccl.cpp", "ftk_simt.cu", "ftk_tc.cu", "ftk_s23.cu", "ftk_nufft.cu", "ftk_capi.cu"]
HEADERS = ["ftk_plan_math.h", "ftk_nccl.h", "ftk_tc_dev.cuh", "ftk_internal.cuh", "ftk_tc.cuh", "ftk_sm100.cuh", "ftk_fft.cuh", os.path.join("..", "..", "include", "ftk.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]
if os.environ.get("FTK_S1_PLO"):  # (experiment) Step-1 modes interleaved in the unit order
    FLAGS += ["-DFTK_S1_PLO=" + os.environ["FTK_S1_PLO"]]
if os.environ.get("FTK_S1_HINT"):  # (experiment) Step-1 L2 cache hints
    FLAGS += ["-DFTK_S1_HINT=" + os.environ["FTK_S1_HINT"]]
if os.environ.get("FTK_S1_GEN16"):  # (experiment) Step-1 generator nodes per step: 16 (1) or 32 (0)
    FLAGS += ["-DFTK_S1_GEN16=" + os.environ["FTK_S1_GEN16"]]
if os.environ.get("FTK_DIAG") == "1":  # wait-cycle counters / trace / FTK_S3_DBG (remove _build/ to switch)
    FLAGS += ["-DFTK_DIAG=1"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, ptxas_verbose: bool = False, force: bool = False) -> str:
    """Compile every source (all of them when force=True, else those newer than their object) and link
    libftk.so."""
    os.makedirs(OUT_DIR, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src + ".o")
        objs.append(o)
        if force or _newer(o, [s, __file__] + hdrs):
            cmd = [NVCC] + ARCH + FLAGS + ["-c", s, "-o", o]
            if src.endswith(".cu"):
                cmd += ["-x", "cu"]
                if ptxas_verbose:
                    cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose or ptxas_verbose:
                sys.stderr.write(r.stderr)
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of libftk.so failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))
