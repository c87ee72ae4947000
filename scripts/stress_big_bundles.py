import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
scene, grid, info, desc = scenes.build("tomo", scale=0.0001)
scene.sources = scene.sources[:3].copy()
scene.source_ids = np.arange(3, dtype=np.int64)
scene.rays_per_source = 4_000_000
t.set_field(grid)
res = {}
for sp in ("1", "0"):
    if sp == "1": os.environ["RAYBOS_SPLIT"] = "1"
    else: os.environ.pop("RAYBOS_SPLIT", None)
    r = t.run_trace(scene, True, True)
    res[sp] = r
    print("split", sp, "landed", r.landed, "emitted", r.report["emitted"], "steps", r.report["total_steps"], "ms", r.report["kernel_ms"], "img sum", r.image.sum(), "hit", r.hit_sum.tolist(), flush=True)
a, b = res["1"], res["0"]
print("image equal", np.array_equal(a.image, b.image), "hit equal", np.array_equal(a.hit_sum, b.hit_sum), "landed equal", np.array_equal(a.landed, b.landed))
print("energy ratio", a.image.sum() / (a.landed.sum() / scene.rays_per_source))
