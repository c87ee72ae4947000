"""In-tree build of libraybos_gpu.so (sm_100a only) and of the oracle checkers.

    python -m paper_1812_05902_b200.build

nvcc cross-compiles sm_100a without a GPU, so this runs anywhere the CUDA 12.9
toolkit is installed.  The .so lands next to this file, so it travels with the
repo snapshot to the GPU box (a JIT cache would not).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libraybos_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(ROOT, "include", "raybos_gpu.h"))
    objs = []
    for src in sorted(os.listdir(CSRC)):
        if not src.endswith((".cu", ".cpp")):
            continue
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [path] + hdrs):
            continue
        flags = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo",
                 f"-I{os.path.join(ROOT, 'include')}"]
        if src.endswith(".cu"):
            flags += ARCH + ["-Xptxas", "-v"]
            if src == "kernels_fp64.cu":      # FP64 validation build: no FMA contraction
                flags += ["-fmad=false"]
        else:
            flags += ["-x", "c++", "-Wno-deprecated-gpu-targets"]
        out = _run([NVCC] + flags + ["-c", path, "-o", obj], verbose)
        if verbose and out.strip():
            print(out)
    if force or _stale(LIB, objs):
        _run([NVCC, "-shared"] + ARCH + objs + ["-o", LIB, "-ldl", "-lpthread"], verbose)
    return LIB


CHECKED_LIB = os.path.join(PKG, "libraybos_gpu_checked.so")


def build_checked_library(verbose: bool = False) -> str:
    """The checked build (csrc/render.cuh RB_CHECKED): the same library with every
    K1 shared/global index range-checked, for tests/test_gpu_checked.py (the
    pool's compute-sanitizer is closed).  Shares the host and FP64 objects."""
    build_library(verbose)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    objs = [os.path.join(BUILD, "capi.cpp.o"), os.path.join(BUILD, "kernels_fp64.cu.o")]
    for src in ("kernels.cu", "kernels_nomedium.cu"):
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, "checked_" + src + ".o")
        objs.append(obj)
        if _stale(obj, [path] + hdrs):
            _run([NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-DRB_CHECKED=1",
                  f"-I{os.path.join(ROOT, 'include')}"] + ARCH + ["-c", path, "-o", obj], verbose)
    if _stale(CHECKED_LIB, objs):
        _run([NVCC, "-shared"] + ARCH + objs + ["-o", CHECKED_LIB, "-ldl", "-lpthread"], verbose)
    return CHECKED_LIB


PEAKS_LIB = os.path.join(PKG, "libraybos_peaks.so")


def build_peaks(verbose: bool = False) -> str:
    """Measurement microbenchmarks (FP32 FFMA, L2 gather) used by bench.py."""
    src = os.path.join(PKG, "tools", "peaks.cu")
    if _stale(PEAKS_LIB, [src]):
        _run([NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared"] + ARCH +
             [src, "-o", PEAKS_LIB], verbose)
    return PEAKS_LIB


FAKE_NCCL_SRC = os.path.join(ROOT, "tests", "fake_nccl", "fake_nccl.cpp")
FAKE_NCCL_LIB = os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so")


def build_fake_nccl(verbose: bool = False) -> str:
    """Test infrastructure: the host-staged NCCL stand-in that lets the
    library's multi-GPU paths run on a one-GPU box (RAYBOS_NCCL_LIB)."""
    if _stale(FAKE_NCCL_LIB, [FAKE_NCCL_SRC]):
        _run([NVCC, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-x", "c++",
              FAKE_NCCL_SRC, "-o", FAKE_NCCL_LIB, "-Wno-deprecated-gpu-targets"], verbose)
    return FAKE_NCCL_LIB


def build_oracle(verbose: bool = False) -> None:
    """Builds oracle/liboracle.so and, where /root/reference exists, oracle/_ref."""
    out = _run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], verbose)
    if verbose:
        print(out)


if __name__ == "__main__":
    v = "-v" in sys.argv
    print(build_library(verbose=v, force="--force" in sys.argv))
    print(build_checked_library(verbose=v))
    print(build_peaks(verbose=v))
    print(build_fake_nccl(verbose=v))
    build_oracle(verbose=v)
