"""Parity numbers of the bench scenes vs the C oracle (the measured side of
tests/test_gpu_bench_scenes.py), one JSON line per scene (dev aid)."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle.oracle import COracle
from paper_1812_05902_b200 import scenes
from paper_1812_05902_b200.engine import GpuTracer
from test_gpu_bench_scenes import CASES, pick_emitters, rel_l2

oracle, tracer = COracle(), GpuTracer(1)
for name, (scale, n_img, n_ray) in CASES.items():
    scene, grid, info, desc = scenes.build(name, scale=scale)
    pick = pick_emitters(scene, n_img)
    scene.source_ids = (np.arange(scene.n_sources, dtype=np.int64) if scene.source_ids is None
                        else scene.source_ids)[pick].copy()
    scene.sources = scene.sources[pick].copy()
    field = oracle.field_from_density(grid) if grid is not None else None
    tracer.set_field(grid)
    rng = np.random.default_rng(11)
    src = np.repeat(np.arange(scene.n_sources), 4 * n_ray)
    ray = rng.integers(0, scene.rays_per_source, src.size).astype(np.int32)
    uv, st, steps = tracer.trace_rays(scene, src, ray, grid is not None)
    ruv, rst, rsteps, _ = oracle.trace_rays(scene, field, src, ray, grid is not None)
    ok = (st == 0) & (rst == 0)
    err = np.abs(uv[ok] - ruv[ok]) / scene.sensor.pitch
    # deflection by the medium: the same rays traced without it
    if grid is not None:
        nuv, nst, _ = tracer.trace_rays(scene, src, ray, False)
        both = ok & (nst == 0)
        defl = np.hypot(*(uv[both] - nuv[both]).T) / scene.sensor.pitch
    else:
        defl = np.zeros(1)
    a = tracer.run_trace(scene, grid is not None, True)
    b = oracle.trace(scene, field, grid is not None, True)
    m = a.landed > 0
    d = np.abs(a.hit_sum[m] / a.landed[m, None] - b.hit_sum[m] / b.landed[m, None]).max()
    print(json.dumps({"scene": name, "emitters": scene.n_sources, "rays_per_emitter": scene.rays_per_source,
                      "rays_sampled": int(src.size), "outcomes_equal": bool(np.array_equal(st, rst)),
                      "ray_err_px_max": float(err.max()), "ray_err_px_rms": float(np.sqrt((err ** 2).mean())),
                      "steps_mean": float(steps[ok].mean()),
                      "deflection_px_max": float(defl.max()), "rays_deflected_gt_0.01px": int((defl > 0.01).sum()), "steps_max_diff": int(np.abs(steps - rsteps).max()),
                      "landed_equal": bool(np.array_equal(a.landed, b.landed)),
                      "mean_hit_err_px": float(d / scene.sensor.pitch),
                      "image_rel_l2": float(rel_l2(a.image, b.image))}), flush=True)
