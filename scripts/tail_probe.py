"""Rays/s of a bench scene for several bundle sizes (dev aid): is the partial
last patch iteration of each emitter (idle warps) visible?"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
name, scale = sys.argv[1], float(sys.argv[2])
t = GpuTracer(1)
scene, grid, info, desc = scenes.build(name, scale=scale)
t.set_field(grid)
for N in [int(x) for x in sys.argv[3:]]:
    scene.rays_per_source = N
    t.run_trace(scene, True, True)
    best = min(t.run_trace(scene, True, True).report["kernel_ms"] for _ in range(3))
    r = t.run_trace(scene, True, True)
    rays = scene.n_sources * N
    print(json.dumps({"scene": name, "N": N, "rays_per_s": rays / best * 1e3,
                      "steps_per_s": r.report["total_steps"] / best * 1e3}))
