"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Each fixture holds, for one scene built by the reference's own
parse_config_json + build_scene_setup (engine.cpp:228-427):
  scene_json  the flat rb_scene (include/raybos_gpu.h) the reference resolved
  field_*     GriddedField node arrays (FP64) when the scene has a medium
  ray_*       per-ray replay of process_source for a sample of (source, ray)
  hit_sum, landed, counters, image   reference run_trace outputs (FP64)
for the traces with_field = 1 and 0.  The GPU parity tests read only these
files (the reference does not exist on the GPU box).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402

THIN = [{"type": "aperture", "f_number": 11},
        {"type": "thin_lens", "focal_length_m": 0.105, "diameter_m": 0.03}]


def cfg(source, medium, optics=THIN, sensor=(128, 128), rays=1000, sampling="stratified", seed=1234,
        extra=None):
    c = {
        "scene": {"source": source, "medium": medium, "gladstone_dale_m3_kg": 2.26e-4,
                  "ambient_rho_kg_m3": 1.225},
        "geometry": {"z_dot_to_volume_m": 0.25, "z_volume_to_lens_m": 0.73},
        "optics": optics,
        "sensor": {"resolution": list(sensor), "pitch_m": 1.0e-5, "bit_depth": 16, "gain": "auto",
                   "distance_m": "auto"},
        "bundle": {"rays_per_source": rays, "sampling": sampling, "seed": seed,
                   "wavelength_m": 5.0e-7},
        "bos": {"magnification": 0.12, "grid_nodes": [5, 5], "grid_extent_m": [0.006, 0.006]},
    }
    if extra:
        for k, v in extra.items():
            c[k].update(v)
    return json.dumps(c)


SLAB = {"type": "uniform_gradient_slab", "rho0_kg_m3": 1.225, "grad_kg_m4": [10, 0],
        "extent_m": [0.048, 0.048], "depth_m": 0.01, "nodes": [25, 25, 5]}
BLOB = {"type": "gaussian_blob_slab", "rho0_kg_m3": 1.225, "amplitude_kg_m3": 2.0,
        "sigma_m": 0.004, "extent_m": [0.032, 0.032], "depth_m": 0.01, "nodes": [65, 65, 3]}
SINGLET = [{"type": "aperture", "f_number": 4},
           {"type": "singlet", "r1_m": 0.103, "r2_m": -0.103, "thickness_m": 0.005,
            "glass_index": 1.5, "diameter_m": 0.06}]
ABERR = [{"type": "aperture", "f_number": 2.8},
         {"type": "singlet", "r1_m": 0.103, "r2_m": -0.103, "thickness_m": 0.005,
          "glass_index": 1.5, "diameter_m": 0.08}]

FIXTURES = {
    # test_engine.cpp:21-31 small_config (bos_uniform scaled down)
    "small": dict(builtin="small"),
    # acceptance null test shape, fewer dots (validate.cpp:387-399)
    "null_small": dict(json=cfg({"type": "dots", "extent_m": [0.02, 0.02], "count": 16, "seed": 5},
                                dict(SLAB, grad_kg_m4=[0, 0], nodes=[9, 9, 5]), rays=2000,
                                seed=21)),
    # strong stacked Gaussian blob slab (bos_blob shape, 4x amplitude): curved trajectories
    "blob": dict(json=cfg({"type": "dots", "extent_m": [0.03, 0.03], "count": 24, "seed": 11},
                          BLOB, sensor=(160, 160), rays=900, seed=99)),
    # non-square bundle, uniform-random sampling (raygen.cpp:57-63 argument order)
    "uniform_random": dict(json=cfg({"type": "dots", "extent_m": [0.01, 0.01], "count": 10,
                                     "seed": 3}, SLAB, sensor=(96, 96), rays=300,
                                    sampling="uniform-random", seed=17)),
    # PIV particles, no medium, thick singlet, out of focus (configs/demo_out_of_focus.json)
    "singlet_defocus": dict(json=cfg({"type": "particles", "count": 40, "diameter_m": 5e-6,
                                      "seed": 9, "box_lo_m": [-0.015, -0.015, -0.02],
                                      "box_hi_m": [0.015, 0.015, 0.02]},
                                     {"type": "none"}, optics=SINGLET, sensor=(256, 256),
                                     rays=500, seed=4)),
    # f/2.8 singlet with spherical aberration (configs/demo_aberration.json)
    "aberration": dict(json=cfg({"type": "dots", "extent_m": [0.06, 0.06], "count": 30,
                                 "seed": 13}, {"type": "none"}, optics=ABERR, sensor=(256, 256),
                                rays=600, seed=6)),
    # genuinely 3-D Gaussian blob (not a stacked slice), ~95 RK4 steps per ray
    "field3d": dict(json=cfg({"type": "dots", "extent_m": [0.02, 0.02], "count": 20, "seed": 31},
                             {"type": "none"}, sensor=(128, 128), rays=700, seed=5),
                    density="blob3d"),
    # Tomo-PIV shape: particles INSIDE a normal-shock volume (ray origins in the box)
    "shock_particles": dict(json=cfg({"type": "particles", "count": 30, "diameter_m": 5e-6,
                                      "seed": 19, "box_lo_m": [-0.005, -0.005, 0.247],
                                      "box_hi_m": [0.005, 0.005, 0.253]},
                                     {"type": "none"}, sensor=(128, 128), rays=800, seed=12),
                            density="shock"),
    # folded camera: aperture + thin lens + a 45-degree plane mirror (reflect_on_mirror,
    # optics.cpp:134-141) turning the beam to +y onto a sensor facing -y, through
    # the Gaussian blob field
    "mirror_fold": dict(json=cfg({"type": "dots", "extent_m": [0.012, 0.012], "count": 20,
                                  "seed": 23}, BLOB, sensor=(160, 160), rays=600, seed=41),
                        camera="fold"),
    # off-axis perspective camera: the whole camera (pupil, thick singlet, sensor
    # frame) turned 14 deg about y and -9 deg about x around the centre of a
    # normal-shock volume, so plane_basis, the singlet's spherical caps and the
    # sensor basis all run with general axes (SceneSetup level, as build_scene_setup
    # only builds +z cameras, engine.cpp:258)
    "tilted_camera": dict(json=cfg({"type": "particles", "count": 24, "diameter_m": 5e-6,
                                    "seed": 29, "box_lo_m": [-0.005, -0.005, 0.247],
                                    "box_hi_m": [0.005, 0.005, 0.253]},
                                   {"type": "none"}, optics=SINGLET, sensor=(160, 160),
                                   rays=700, sampling="uniform-random", seed=37),
                          density="shock", camera="tilt"),
    # single-ray bundles (raygen.cpp:45-46) and the 15.03 um spot convention
    "single_ray": dict(json=cfg({"type": "dots", "extent_m": [0.01, 0.01], "count": 50,
                                 "seed": 2}, SLAB, sensor=(96, 96), rays=1, seed=8,
                                extra={"sensor": {"diffraction_pi_factor": False}})),
}


def density(kind):
    """Synthetic DensityVolume (scene.hpp:25-40) centred at z = Z_D = 0.25 m."""
    from paper_1812_05902_b200.scene import DensityGrid
    if kind == "blob3d":
        n, ext = 48, 0.016
        sp = ext / (n - 1)
        c = (np.arange(n) * sp - 0.5 * ext)
        z, y, x = np.meshgrid(c, c, c, indexing="ij")
        rho = 1.225 + 5.0 * np.exp(-(x * x + y * y + z * z) / (2 * 0.003 ** 2))
        g = DensityGrid(n, n, n, (-0.5 * ext, -0.5 * ext, 0.25 - 0.5 * ext), (sp, sp, sp),
                        rho.astype(np.float32).ravel())
    else:  # normal shock, rho2/rho1 = 2.667 (M = 2), thickness ~2 cells
        nx, ny, nz = 48, 48, 24
        ext = (0.012, 0.012, 0.008)
        sp = tuple(e / (k - 1) for e, k in zip(ext, (nx, ny, nz)))
        x = np.arange(nx) * sp[0] - 0.5 * ext[0]
        rho_x = 1.225 + (2.667 - 1.0) * 1.225 * 0.5 * (1 + np.tanh(x / (2 * sp[0])))
        rho = np.broadcast_to(rho_x, (nz, ny, nx))
        g = DensityGrid(nx, ny, nz, (-0.5 * ext[0], -0.5 * ext[1], 0.25 - 0.5 * ext[2]), sp,
                        np.ascontiguousarray(rho, dtype=np.float32).ravel())
    h = 0.5 * min(g.spacing)
    lo, hi = g.bounds()
    return g, h, int(4.0 * np.linalg.norm(hi - lo) / h) + 64


def move_camera(scene, kind):
    """SceneSetup-level cameras the reference's config schema cannot express."""
    from paper_1812_05902_b200 import abi
    from paper_1812_05902_b200.scene import plane_mirror, rotation
    if kind == "tilt":
        rot = rotation((1.0, 0.0, 0.0), -9.0) @ rotation((0.0, 1.0, 0.0), 14.0)
        return scene.with_camera_moved(rot, (0.0, 0.0, 0.25))
    # fold: mirror 40 mm behind the lens, normal (0, 1, -1)/sqrt(2); everything the
    # beam meets after it (the sensor) is reflected through the mirror plane
    lens_z = max(e.center.z for e in scene.elements)
    m = np.array([0.0, 0.0, lens_z + 0.04])
    n = np.array([0.0, 1.0, -1.0]) / np.sqrt(2.0)
    H = np.eye(3) - 2.0 * np.outer(n, n)

    def refl_pt(v):
        return abi.vec3(H @ (np.array([v.x, v.y, v.z]) - m) + m)

    def refl_ax(v):
        return abi.vec3(H @ np.array([v.x, v.y, v.z]))

    se = scene.sensor
    scene.elements = list(scene.elements) + [plane_mirror(m, n, 0.06)]
    scene.sensor = abi.Sensor(refl_pt(se.center), refl_ax(se.normal), refl_ax(se.e_u),
                              refl_ax(se.e_v), se.width_px, se.height_px, se.pitch,
                              se.window_sigmas)
    return scene


def make(name, spec, n_ray_samples=2048):
    ref = Reference(json_text=spec.get("json"), builtin=spec.get("builtin"))
    if spec.get("density"):
        grid, h, max_steps = density(spec["density"])
        ref.set_field_density(grid)
        ref.lib().refshim_set_step(ref.h, h, max_steps)
    if spec.get("camera"):
        ref.set_flat(move_camera(ref.scene(), spec["camera"]))
    scene = ref.scene()
    if spec.get("density"):
        out_rho = {"field_rho": grid.rho, "field_k": np.array(grid.gladstone_dale)}
    else:
        out_rho = {}
    field = ref.field()
    info = ref.info()
    out = {"scene_json": np.array(json.dumps(scene.to_json())), **out_rho}
    if field is not None:
        out.update(field_dims=np.array([field.nx, field.ny, field.nz]),
                   field_origin=np.array(field.origin), field_spacing=np.array(field.spacing),
                   field_n=field.n, field_gx=field.gx, field_gy=field.gy, field_gz=field.gz)
    rng = np.random.default_rng(0)
    n = scene.n_sources * scene.rays_per_source
    pick = np.sort(rng.choice(n, size=min(n, n_ray_samples), replace=False))
    src = (pick // scene.rays_per_source).astype(np.int64)
    ray = (pick % scene.rays_per_source).astype(np.int32)
    out["ray_src"], out["ray_idx"] = src, ray
    out["info"] = np.array([info.magnification, info.f_number, info.gain, info.d_tau,
                            info.lens_plane_z, info.focal_length])
    if field is not None:  # trace_debug records for a few rays (engine.cpp:605-624)
        dbg = [(0, 0), (scene.n_sources // 2, scene.rays_per_source // 2),
               (scene.n_sources - 1, scene.rays_per_source - 1)]
        out["debug_rays"] = np.array(dbg, dtype=np.int64)
        for k, (d_, r_) in enumerate(dbg):
            out[f"debug_{k}"] = ref.trace_debug(d_, r_)
    for wf in (1, 0):
        uv, status, steps, exit_state = ref.trace_rays(src, ray, with_field=bool(wf))
        out[f"ray_uv_{wf}"], out[f"ray_status_{wf}"], out[f"ray_steps_{wf}"] = uv, status, steps
        res = ref.run_trace(with_field=bool(wf), accumulate_image=True, threads=0)
        r = res.report
        out[f"hit_sum_{wf}"] = res.hit_sum
        out[f"landed_{wf}"] = res.landed
        out[f"counters_{wf}"] = np.array([r["emitted"], r["landed"], r["lost"],
                                          r["blocked_aperture"], r["blocked_miss"],
                                          r["blocked_tir"], r["blocked_sensor_miss"]])
        out[f"image_{wf}"] = res.image
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    return path, os.path.getsize(path)


if __name__ == "__main__":
    names = sys.argv[1:] or list(FIXTURES)
    for nm in names:
        p, sz = make(nm, FIXTURES[nm])
        print(f"{nm}: {sz / 1024:.0f} KB -> {p}")
