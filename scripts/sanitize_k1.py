"""Small K1 workload for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python scripts/sanitize_k1.py [fixture ...]

Renders the committed golden fixtures through every K1 entry point the bench
and the drop-in use — rb_trace with the image (shared-memory tile, work queue,
split-emitter partials), rb_trace_bos_pair, rb_trace_rays — with the emitter
split forced to several values so the chunk-partial path runs too.  Each result
is checked against the oracle so a sanitizer run that passes also proves the
instrumented binary still computes the right answer.  SURVEY §5.2; replaces the
reference's race-freedom-by-construction contract (engine.cpp:442-447).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def main(names):
    from golden_io import load
    from oracle.oracle import COracle
    from paper_1812_05902_b200.engine import GpuTracer
    orc = COracle()
    with GpuTracer(n_devices=1) as t:
        for name in names:
            scene, field, g = load(name)
            ref = orc.trace(scene, field, True, True)
            t.set_field(field)
            for split in ("1", "3"):
                os.environ["RAYBOS_SPLIT"] = split
                res = t.run_trace(scene, with_field=True, accumulate_image=True)
                assert np.array_equal(res.landed, ref.landed), (name, split)
                rel = np.linalg.norm(res.image - ref.image) / max(np.linalg.norm(ref.image), 1e-300)
                assert rel < 1e-4, (name, split, rel)
            os.environ.pop("RAYBOS_SPLIT", None)
            if field is not None:
                r0, r1 = t.trace_bos_pair(scene)
                assert np.array_equal(r1.landed, ref.landed), name
            n = min(scene.n_sources * scene.rays_per_source, 512)
            src = np.arange(n) % scene.n_sources
            ray = (np.arange(n) * 7) % scene.rays_per_source
            t.trace_rays(scene, src, ray, with_field=True)
            print(f"{name}: ok ({scene.n_sources} x {scene.rays_per_source} rays)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["small", "blob"])
