import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from golden_io import load
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
for name in ["small", "aberration"]:
    scene, field, g = load(name)
    t.set_field(field)
    uv, st, steps = t.trace_rays_fp64(scene, g["ray_src"], g["ray_idx"], False)
    ref = g["ray_uv_0"]
    ok = st == 0
    neq = ~np.all(uv == ref, axis=1) & ok
    print(name, "mismatch", neq.sum(), "of", ok.sum())
    idx = np.where(neq)[0][:5]
    for q in idx:
        print(q, g["ray_src"][q], g["ray_idx"][q], uv[q].tolist(), ref[q].tolist(), (uv[q] - ref[q]).tolist())
    # stats for the sources involved
    res = t.trace_stats_fp64(scene, False)
    print("stats equal (wf=0)", np.array_equal(res.hit_sum, g["hit_sum_0"]))
