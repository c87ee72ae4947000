"""Builds launch-configuration variants of libraybos_gpu.so for A/B timing (dev aid)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1812_05902_b200")
OUT = os.path.join(PKG, "_variants")
os.makedirs(OUT, exist_ok=True)
NVCC = "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
capi = os.path.join(PKG, "_build", "capi.cpp.o")
fp64 = os.path.join(PKG, "_build", "kernels_fp64.cu.o")
variants = []
for v in sys.argv[1:] or ["256x2c1", "256x3c0"]:
    b, rest = v.split("x")
    u, dd, sp, ur = 1, 1, 0, 1
    if "r" in rest:
        rest, ur = rest.split("r")
    if "s" in rest:
        rest, sp = rest.split("s")
    if "d" in rest:
        rest, dd = rest.split("d")
    if "u" in rest:
        rest, u = rest.split("u")
    m, c = rest.split("c") if "c" in rest else (rest, "1")
    variants.append((int(b), int(m), int(c), int(u), int(dd), int(sp), int(ur)))
for blk, mb, cc, uu, dd, sp, ur in variants:
    tag = os.environ.get("TAG", "")
    obj = os.path.join(OUT, f"k_{blk}_{mb}_c{cc}_u{uu}_d{dd}_s{sp}_r{ur}{tag}.o")
    subprocess.run([NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", *ARCH,
                    f"-DRB_BLOCK={blk}", f"-DRB_MINB={mb}", f"-DRB_UNIFORM_RELOAD={uu}", f"-DRB_DITHER={dd}", f"-DRB_STEP_UNROLL={ur}", *os.environ.get("EXTRA", "").split(), f"-I{ROOT}/include", "-c",
                    os.path.join(PKG, "csrc", "kernels.cu"), "-o", obj], check=True)
    lib = os.path.join(OUT, f"libraybos_gpu_{blk}_{mb}_c{cc}_u{uu}_d{dd}_s{sp}_r{ur}{tag}.so")
    subprocess.run([NVCC, "-shared", *ARCH, capi, fp64, obj, "-o", lib, "-ldl", "-lpthread"], check=True)
    print(lib)
