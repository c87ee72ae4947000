"""render_warps vs render_emitters (dev aid): bit-identical outputs on every
field fixture and bench scene sample, then rays/s of both."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from golden_io import NAMES, load
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
def both(scene):
    os.environ.pop("RAYBOS_K1", None)
    a = t.run_trace(scene)
    os.environ["RAYBOS_K1"] = "warp"
    b = t.run_trace(scene)
    os.environ.pop("RAYBOS_K1", None)
    return a, b
for name in NAMES:
    scene, field, g = load(name)
    if field is None:
        continue
    t.set_field(field)
    a, b = both(scene)
    ok = (np.array_equal(a.image, b.image) and np.array_equal(a.hit_sum, b.hit_sum) and
          np.array_equal(a.landed, b.landed) and a.report["total_steps"] == b.report["total_steps"]
          and a.report["lost"] == b.report["lost"])
    print(name, "identical" if ok else "DIFFER", flush=True)
    assert ok
for name, scale in (("tomo", 0.1), ("bos", 0.05), ("large", 0.002)):
    scene, grid, info, desc = scenes.build(name, scale=scale)
    t.set_field(grid)
    a, b = both(scene)
    assert np.array_equal(a.image, b.image) and np.array_equal(a.hit_sum, b.hit_sum)
    res = {}
    for mode in ("cta", "warp"):
        if mode == "warp":
            os.environ["RAYBOS_K1"] = "warp"
        else:
            os.environ.pop("RAYBOS_K1", None)
        t.run_trace(scene)
        best = min(t.run_trace(scene).report["kernel_ms"] for _ in range(3))
        res[mode] = scene.n_sources * scene.rays_per_source / best * 1e3
    os.environ.pop("RAYBOS_K1", None)
    print(json.dumps({"scene": name, "identical": True, **{k: f"{v:.4g}" for k, v in res.items()},
                      "gain": res["warp"] / res["cta"] - 1}), flush=True)
