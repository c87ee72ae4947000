"""Runs K1's entry points through the bounds-checked library (RAYBOS_LIB =
libraybos_gpu_checked.so, csrc/render.cuh RB_CHECKED) on every golden fixture
and on the bench scenes at reduced emitter counts, and prints one JSON line per
case with what the calls returned.  A range violation inside K1 makes the call
fail with "checked build: ..." (tests/test_gpu_checked.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def run(t, name, scene, field, out):
    t.set_field(field)
    rec = {"case": name}
    for split in ("1", "3"):
        os.environ["RAYBOS_SPLIT"] = split
        res = t.run_trace(scene, with_field=True, accumulate_image=True)
        rec[f"landed_split{split}"] = int(res.landed.sum())
        rec[f"image_sum_split{split}"] = float(res.image.sum())
    os.environ.pop("RAYBOS_SPLIT", None)
    if field is not None:
        r0, r1 = t.trace_bos_pair(scene)
        rec["pair_landed"] = int(r1.landed.sum())
    n = min(scene.n_sources * scene.rays_per_source, 4096)
    src = np.arange(n) % scene.n_sources
    ray = (np.arange(n) * 7919) % scene.rays_per_source
    uv, st, steps = t.trace_rays(scene, src, ray, with_field=True)
    rec["rays_landed"] = int((st == 0).sum())
    out.write(json.dumps(rec) + "\n")
    out.flush()


def main():
    from golden_io import NAMES, load
    from paper_1812_05902_b200 import abi, scenes
    from paper_1812_05902_b200.engine import GpuTracer
    assert os.path.basename(abi.load_library()._name) == "libraybos_gpu_checked.so"
    with GpuTracer(1) as t:
        for name in NAMES:
            scene, field, g = load(name)
            run(t, name, scene, field, sys.stdout)
            # wide (>12 px) and degenerate spots: the other deposit paths
            for k, scale in (("wide", 3.0), ("degenerate", 1e-4)):
                s2 = scene.subset(np.arange(min(scene.n_sources, 6)))
                s2.d_tau = scene.d_tau * scale
                run(t, f"{name}/{k}", s2, field, sys.stdout)
        for name, scale in (("piv", 1.0), ("optics", 0.01), ("tomo", 0.005), ("bos", 0.02),
                            ("large", 0.0005)):
            scene, grid, info, desc = scenes.build(name, scale=scale)
            run(t, f"bench/{name}", scene, grid, sys.stdout)


if __name__ == "__main__":
    main()
