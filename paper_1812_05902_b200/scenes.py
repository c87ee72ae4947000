"""Synthetic scenes of the five BASELINE.json shapes.

Each builder returns a reference-schema config (the JSON keys of
proj/src/config.cpp:109-196) plus an in-memory density volume, resolved with
:func:`paper_1812_05902_b200.setup.build_scene` exactly like the reference's
build_scene_setup would resolve the same config with a GVOL medium.  All data
are synthetic and seeded; nothing is downloaded.

  piv     1e3 particles x 1e3 rays, no medium, thin lens, 512^2
  bos     20,480 dots x 1e4 rays through a 256^3 BDT-like field (64 mm cube), 1024^2
  tomo    1e5 particles x 1e4 rays (1e9) inside a 256x256x128 normal-shock field,
          thick singlet camera, 2048^2                                  <- headline
  optics  1e4 particles x 1e4 rays, f/2.8 singlet, +-20 mm depth, off-axis perspective
          camera (turned 20 deg / 6 deg about the box centre), 1024^2
  large   4e5 dots x 1e4 rays through a 1024^3 grid (16 GiB float4), 4096^2, fine
          step (h = spacing / 4, half the reference default)
"""
from __future__ import annotations

import math

import numpy as np

from . import setup as S
from .scene import DensityGrid

THIN = [{"type": "aperture", "f_number": 11},
        {"type": "thin_lens", "focal_length_m": 0.105, "diameter_m": 0.03}]
SINGLET_F11 = [{"type": "aperture", "f_number": 11},
               {"type": "singlet", "r1_m": 0.103, "r2_m": -0.103, "thickness_m": 0.005,
                "glass_index": 1.5, "diameter_m": 0.03}]
SINGLET_F28 = [{"type": "aperture", "f_number": 2.8},
               {"type": "singlet", "r1_m": 0.103, "r2_m": -0.103, "thickness_m": 0.005,
                "glass_index": 1.5, "diameter_m": 0.08}]


def _cfg(source, sensor, rays, optics, seed=1234, magnification=None, distance="auto",
         delta_xi=0.0):
    c = {"scene": {"source": source, "medium": {"type": "none"},
                   "gladstone_dale_m3_kg": 2.26e-4, "ambient_rho_kg_m3": 1.225},
         "geometry": {"z_dot_to_volume_m": 0.25, "z_volume_to_lens_m": 0.73},
         "optics": optics,
         "sensor": {"resolution": list(sensor), "pitch_m": 1e-5, "bit_depth": 16, "gain": "auto",
                    "distance_m": distance},
         "bundle": {"rays_per_source": rays, "sampling": "stratified", "seed": seed,
                    "wavelength_m": 5e-7},
         "trace": {"delta_xi_m": delta_xi},
         "bos": {}}
    if magnification:
        c["bos"]["magnification"] = magnification
    return c


def bdt_field(n_xy: int, n_z: int, extent_xy: float, depth: float, modes: int = 24,
              amplitude: float = 0.05, seed: int = 7) -> DensityGrid:
    """Buoyancy-driven-turbulence-like density: random-phase Fourier modes in
    (x, y) about rho0 = 1.225 kg/m^3, stacked in z (paper section 4)."""
    rng = np.random.default_rng(seed)
    x = np.linspace(-0.5 * extent_xy, 0.5 * extent_xy, n_xy)
    X, Y = np.meshgrid(x, x, indexing="xy")
    rho = np.full((n_xy, n_xy), 1.225)
    L = extent_xy
    for _ in range(modes):
        kx, ky = rng.integers(1, 9, size=2) * rng.choice([-1, 1], size=2)
        a = amplitude / math.sqrt(modes) * rng.uniform(0.5, 1.5) / math.hypot(kx, ky) ** 0.5
        rho += a * np.cos(2 * np.pi * (kx * X + ky * Y) / L + rng.uniform(0, 2 * np.pi))
    sl = rho.astype(np.float32).ravel()
    dx = extent_xy / (n_xy - 1)
    dz = depth / (n_z - 1)
    return DensityGrid(n_xy, n_xy, n_z, (-0.5 * extent_xy, -0.5 * extent_xy, 0.0), (dx, dx, dz),
                       np.tile(sl, n_z))


def shock_field(nx: int, ny: int, nz: int, ext, delta_cells: float = 2.0,
                ratio: float = 2.667) -> DensityGrid:
    """Normal shock (M = 2, gamma = 1.4): rho1 + (rho2 - rho1) * (1 + tanh(x / delta)) / 2."""
    sp = tuple(e / (k - 1) for e, k in zip(ext, (nx, ny, nz)))
    x = np.arange(nx) * sp[0] - 0.5 * ext[0]
    rho1 = 1.225
    rho_x = rho1 + (ratio - 1.0) * rho1 * 0.5 * (1.0 + np.tanh(x / (delta_cells * sp[0])))
    rho = np.broadcast_to(rho_x.astype(np.float32), (nz, ny, nx))
    return DensityGrid(nx, ny, nz, (-0.5 * ext[0], -0.5 * ext[1], -0.5 * ext[2]), sp,
                       np.ascontiguousarray(rho).ravel())


def _focus_on(cfg: dict, z_obj: float) -> tuple:
    """Sensor distance (from the last element) and magnification that focus the
    camera on the plane z = z_obj instead of the target plane z = 0."""
    c = S.parse_config(dict(cfg, sensor=dict(cfg["sensor"], gain=1.0, distance_m=0.05)))
    scene, _, info = S.build_scene(c)
    h = 0.05 * scene.pupil_radius
    pz = scene.pupil_center[2]
    probes = []
    for sign in (1.0, -1.0):
        o, d, r = S.propagate_chain((0.0, 0.0, z_obj), S._normalized((sign * h, 0.0, pz - z_obj)),
                                    scene.elements)
        assert r == 0
        probes.append((o, d))
    (ao, ad), (bo, bd) = probes
    sa, sb = ad[0] / ad[2], bd[0] / bd[2]
    z_img = (bo[0] - ao[0] + sa * ao[2] - sb * bo[2]) / (sa - sb)
    last = max(e.back.vertex.z if e.kind == 1 else e.center.z for e in scene.elements)
    # chief ray from a small off-axis point of the object plane -> magnification
    xt = 2e-4
    o, d, r = S.propagate_chain((xt, 0.0, z_obj), S._normalized((-xt, 0.0, pz - z_obj)),
                                scene.elements)
    t = (z_img - o[2]) / d[2]
    mag = abs(o[0] + d[0] * t) / xt
    return z_img - last, mag


def config(name: str, scale: float = 1.0):
    """Returns (config dict, DensityGrid | None, description dict)."""
    if name == "piv":
        cfg = _cfg({"type": "particles", "count": int(1000 * scale), "diameter_m": 5e-6, "seed": 9,
                    "box_lo_m": [-0.015, -0.015, -0.002], "box_hi_m": [0.015, 0.015, 0.002]},
                   (512, 512), 1000, THIN, magnification=0.12)
        return cfg, None, {"emitters": int(1000 * scale), "rays_per_emitter": 1000}
    if name == "bos":
        ext = 1024 * 1e-5 / 0.12
        cfg = _cfg({"type": "dots", "extent_m": [ext, ext], "density_per_32px_region": 20 * scale,
                    "seed": 7}, (1024, 1024), 10000, THIN, magnification=0.12)
        grid = bdt_field(256, 256, 0.064, 0.064)
        return cfg, grid, {"field": "256^3 BDT-like, 64 mm cube"}
    if name == "tomo":
        n_src = int(100000 * scale)
        cfg = _cfg({"type": "particles", "count": n_src, "diameter_m": 5e-6, "seed": 9,
                    "box_lo_m": [-0.06, -0.06, 0.244], "box_hi_m": [0.06, 0.06, 0.256]},
                   (2048, 2048), 10000, SINGLET_F11, delta_xi=1e-4)
        dist, mag = _focus_on(cfg, 0.25)
        cfg["sensor"]["distance_m"] = dist
        cfg["bos"]["magnification"] = mag
        grid = shock_field(256, 256, 128, (0.128, 0.128, 0.032))
        return cfg, grid, {"field": "256x256x128 normal shock, 128x128x32 mm", "emitters": n_src}
    if name == "optics":
        n_src = int(10000 * scale)
        cfg = _cfg({"type": "particles", "count": n_src, "diameter_m": 5e-6, "seed": 13,
                    "box_lo_m": [-0.01, -0.03, -0.02], "box_hi_m": [0.03, 0.03, 0.02]},
                   (1024, 1024), 10000, SINGLET_F28, seed=6)
        return cfg, None, {"emitters": n_src, "camera": OPTICS_CAMERA}
    if name == "large":
        ext = 4096 * 1e-5 / 0.12
        n_src = int(400000 * scale)
        # BASELINE's "fine integration step": half the reference default
        # (engine.cpp:244-252 takes h = spacing / 2), i.e. h = spacing / 4
        h = 0.25 * 0.256 / 1023
        cfg = _cfg({"type": "dots", "extent_m": [ext, ext], "count": n_src, "seed": 17},
                   (4096, 4096), 10000, THIN, magnification=0.12, delta_xi=h)
        grid = bdt_field(1024, 1024, 0.256, 0.256, amplitude=0.1)
        return cfg, grid, {"field": "1024^3 BDT-like, 256 mm cube, fine step h = spacing/4"}
    raise ValueError(f"unknown scene '{name}'")


# The optics scene's off-axis perspective camera (BASELINE configs[3]): the
# whole +z camera build_scene_setup makes (pupil, f/2.8 singlet, sensor frame)
# turned 20 deg about y and 6 deg about x around the particle box's centre, so
# the box is seen obliquely (perspective foreshortening, depth-varying defocus)
# and every optical axis is general.
OPTICS_CAMERA = {"pivot": (0.01, 0.0, 0.0), "rot_y_deg": 20.0, "rot_x_deg": 6.0}


def build(name: str, calibrate=None, scale: float = 1.0):
    """Resolved (FlatScene, DensityGrid | None, SetupInfo, description)."""
    cfg, grid, desc = config(name, scale)
    c = S.parse_config(cfg)
    c.density = grid
    if grid is not None:
        c.medium["depth"] = (grid.nz - 1) * grid.spacing[2]
    if calibrate is None:
        c.sensor["gain"] = 1.0
    scene, field, info = S.build_scene(c, calibrate=calibrate)
    cam = desc.get("camera")
    if cam:  # SceneSetup-level camera move (the gain was calibrated on the +z camera)
        from .scene import rotation
        rot = rotation((1.0, 0.0, 0.0), cam["rot_x_deg"]) @ rotation((0.0, 1.0, 0.0),
                                                                     cam["rot_y_deg"])
        scene = scene.with_camera_moved(rot, cam["pivot"])
        desc = dict(desc, camera=f"off-axis perspective: camera turned {cam['rot_y_deg']} deg "
                                 f"about y, {cam['rot_x_deg']} deg about x around "
                                 f"{cam['pivot']}")
    return scene, field, info, desc
