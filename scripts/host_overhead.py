"""Host-side cost of one rb_trace call on a small scene (dev aid):
python wall per call vs the library's own wall_seconds vs K1 time."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
name = sys.argv[1] if len(sys.argv) > 1 else "piv"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
t = GpuTracer(1)
scene, grid, info, desc = scenes.build(name, scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
t.set_field(grid)
img = torch.zeros(scene.width * scene.height, dtype=torch.int64, device="cuda")
for host_image in (False, True):
    for _ in range(min(20, reps)):
        t.run_trace(scene, True, True, host_image=host_image, image_fixed_ptr=img.data_ptr())
    py, lib, ker = [], [], []
    for _ in range(reps):
        s0 = time.perf_counter()
        r = t.run_trace(scene, True, True, host_image=host_image, image_fixed_ptr=img.data_ptr())
        py.append(time.perf_counter() - s0)
        lib.append(r.report["wall_seconds"])
        ker.append(r.report["kernel_ms"] * 1e-3)
    med = lambda a: float(np.median(a)) * 1e6
    print(f"{name} host_image={host_image}: python {med(py):.1f} us, library {med(lib):.1f} us, "
          f"K1 {med(ker):.1f} us")
s0 = time.perf_counter()
for _ in range(reps):
    sc, keep = scene.to_c()
print(f"to_c {1e6 * (time.perf_counter() - s0) / reps:.1f} us")
