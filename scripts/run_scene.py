"""Renders one bench scene twice (warm-up + measured) — the ncu target (dev aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
name, scale = sys.argv[1], float(sys.argv[2])
t = GpuTracer(1)
scene, grid, info, desc = scenes.build(name, scale=scale)
t.set_field(grid)
for _ in range(2):
    r = t.run_trace(scene, True, True)
rays = scene.n_sources * scene.rays_per_source
print(name, rays, r.report["kernel_ms"], rays / r.report["kernel_ms"] * 1e3, r.report["total_steps"] / rays)
