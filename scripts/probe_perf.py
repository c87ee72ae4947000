"""Quick throughput probe on golden-fixture geometry (development aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from golden_io import load
from paper_1812_05902_b200.engine import GpuTracer

t = GpuTracer(1)
for name, n_src, rays in [("field3d", 2000, 10000), ("blob", 2000, 10000), ("singlet_defocus", 2000, 10000), ("small", 2000, 10000)]:
    scene, field, g = load(name)
    rng = np.random.default_rng(1)
    lo = scene.sources.min(0); hi = scene.sources.max(0)
    scene.sources = rng.uniform(lo, hi, size=(n_src, 3))
    scene.rays_per_source = rays
    t.set_field(field)
    for wf in (1,):
        t.run_trace(scene, bool(wf), True)
        ts = []
        for _ in range(3):
            r = t.run_trace(scene, bool(wf), True)
            ts.append(r.report["kernel_ms"])
        ms = min(ts)
        rays_tot = n_src * rays
        print(f"{name:16s} wf={wf} rays={rays_tot:.2e} steps/ray={r.report['total_steps']/rays_tot:6.1f} "
              f"kernel {ms:8.3f} ms  {rays_tot/ms*1e3:.3e} rays/s  wall {r.report['wall_seconds']*1e3:.1f} ms", flush=True)
