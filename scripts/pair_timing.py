"""bos_run's two traces: fused pair kernel vs two separate traces (dev aid)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
scene, grid, info, desc = scenes.build("bos", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 0.05)
t.set_field(grid)
for _ in range(2):
    a = t.run_trace(scene, False, False); b = t.run_trace(scene, True, False); p = t.trace_bos_pair(scene)
two = a.report["kernel_ms"] + b.report["kernel_ms"]
print("rays", scene.n_sources * scene.rays_per_source, "two traces ms %.2f (no field %.2f + field %.2f)" % (two, a.report["kernel_ms"], b.report["kernel_ms"]),
      "pair ms %.2f" % p[1].report["kernel_ms"])
