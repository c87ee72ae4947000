"""Checks the 1024^3 cell table against the node path on sampled rays (dev aid)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
scene, grid, info, desc = scenes.build("large", scale=0.002)
rng = np.random.default_rng(3)
src = rng.integers(0, scene.n_sources, 4096)
ray = rng.integers(0, scene.rays_per_source, 4096).astype(np.int32)
out = {}
for flag in ("1", "0"):
    os.environ["RAYBOS_CELL_TABLE"] = flag
    t0 = time.perf_counter(); t.set_field(grid); dt = time.perf_counter() - t0
    uv, st, steps = t.trace_rays(scene, src, ray, True)
    out[flag] = (uv, st, steps)
    print("table", flag, "set_field s %.2f" % dt, "field GB %.1f" % (t.field_bytes() / 1e9), flush=True)
    uv0, st0, _ = t.trace_rays(scene, src, ray, False)
    ok = (st == 0) & (st0 == 0)
    print("  deflection px max %.4f mean %.4f" % (np.abs(uv[ok] - uv0[ok]).max() / scene.sensor.pitch,
                                               np.abs(uv[ok] - uv0[ok]).mean() / scene.sensor.pitch))
a, b = out["1"], out["0"]
print("status equal", np.array_equal(a[1], b[1]), "uv equal", np.array_equal(a[0], b[0], equal_nan=True),
      "max diff px", np.nanmax(np.abs(a[0] - b[0])) / scene.sensor.pitch)
