"""paper_1812_05902_b200 — B200-native drop-in for the raybos ``run_trace`` hot path.

The product is the C-ABI library ``libraybos_gpu.so`` (include/raybos_gpu.h,
CUDA sm_100a kernels in csrc/).  This package only holds the ctypes mirror of
that ABI (abi.py), scene containers (scene.py), the Python handle on a context
(engine.py), synthetic scene builders for the benchmark configurations
(scenes.py) and the build recipe (build.py).
"""
from .scene import DensityGrid, FieldNodes, FlatScene, TraceResult  # noqa: F401

__all__ = ["DensityGrid", "FieldNodes", "FlatScene", "TraceResult", "GpuTracer", "plan_shards"]


def __getattr__(name):
    if name in ("GpuTracer", "plan_shards", "RaybosError"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
