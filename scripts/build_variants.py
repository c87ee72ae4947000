"""Builds variants of libraybos_gpu.so for A/B timing (dev aid).

usage: EXTRA="-DRB_MINB_CELLS=2 ..." TAG=_x python scripts/build_variants.py
Recompiles kernels.cu with the extra defines (RB_BLOCK, RB_MINB, RB_MINB_CELLS,
RB_MINB_NOFIELD, RB_UNIFORM_RELOAD, RB_DITHER, RB_STEP_UNROLL, RB_MAX_SPOT ...)
and links it with the other current objects of paper_1812_05902_b200/_build
into paper_1812_05902_b200/_variants/libraybos_gpu<TAG>.so."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1812_05902_b200")
OUT = os.path.join(PKG, "_variants")
NVCC = "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

os.makedirs(OUT, exist_ok=True)
tag = os.environ.get("TAG", "_variant")
objs = []
for src in ("kernels.cu", "kernels_nomedium.cu"):   # both K1 translation units
    obj = os.path.join(OUT, f"{src[:-3]}{tag}.o")
    subprocess.run([NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", *ARCH,
                    *os.environ.get("EXTRA", "").split(), f"-I{ROOT}/include", "-c",
                    os.path.join(PKG, "csrc", src), "-o", obj], check=True)
    objs.append(obj)
lib = os.path.join(OUT, f"libraybos_gpu{tag}.so")
others = [os.path.join(PKG, "_build", f) for f in ("capi.cpp.o", "kernels_fp64.cu.o")]
subprocess.run([NVCC, "-shared", *ARCH, *others, *objs, "-o", lib, "-ldl", "-lpthread"], check=True)
print(lib)
