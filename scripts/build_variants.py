"""Builds launch-configuration variants of libraybos_gpu.so for A/B timing (dev aid)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1812_05902_b200")
OUT = os.path.join(PKG, "_variants")
os.makedirs(OUT, exist_ok=True)
NVCC = "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
capi = os.path.join(PKG, "_build", "capi.cpp.o")
variants = [tuple(int(x) for x in v.split("x")) for v in (sys.argv[1:] or ["256x2", "256x3", "256x4", "128x6", "128x8"])]
for blk, mb in variants:
    obj = os.path.join(OUT, f"k_{blk}_{mb}.o")
    subprocess.run([NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", *ARCH,
                    f"-DRB_BLOCK={blk}", f"-DRB_MINB={mb}", f"-I{ROOT}/include", "-c",
                    os.path.join(PKG, "csrc", "kernels.cu"), "-o", obj], check=True)
    lib = os.path.join(OUT, f"libraybos_gpu_{blk}_{mb}.so")
    subprocess.run([NVCC, "-shared", *ARCH, capi, obj, "-o", lib, "-ldl", "-lpthread"], check=True)
    print(lib)
