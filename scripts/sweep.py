"""Times K1 for each library variant on the bench scenes (dev aid).
usage: python scripts/sweep.py <lib.so> [scene scale ...]"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["RAYBOS_LIB"] = sys.argv[1]
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
args = sys.argv[2:] or ["tomo", "0.1", "bos", "0.05", "piv", "1", "optics", "0.1"]
t = GpuTracer(1)
res = {"lib": os.path.basename(sys.argv[1])}
for name, scale in zip(args[0::2], args[1::2]):
    scene, grid, info, desc = scenes.build(name, scale=float(scale))
    t.set_field(grid)
    t.run_trace(scene, True, True)
    best = 1e30
    for _ in range(3):
        r = t.run_trace(scene, True, True)
        best = min(best, r.report["kernel_ms"])
    rays = scene.n_sources * scene.rays_per_source
    spr = r.report["total_steps"] / rays
    res[name] = {"rays_per_s": rays / best * 1e3, "kernel_ms": best, "steps_per_ray": spr,
                 "tflops": (360 * r.report["total_steps"] + 700 * rays) / best * 1e-9}
print(json.dumps(res), flush=True)
