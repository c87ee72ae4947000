"""Config -> scene resolution: the host-side layer ABOVE the drop-in boundary.

Mirrors the reference's ``parse_config_json`` (proj/src/config.cpp:109-196),
``ExperimentConfig::validate`` (config.cpp:206-247) and ``build_scene_setup``
(proj/src/engine.cpp:228-427) so that a reference JSON config (e.g.
proj/configs/*.json) resolves to the same ``FlatScene`` the reference's
SceneSetup flattens to.  This is setup code (a handful of probe rays through
the optics in FP64, the dot/particle generators, the medium volume) — it is
not the hot path and never traces a bundle; the gain calibration dot is
rendered on the GPU through the C-ABI (``calibrate`` callback).

Python floats are IEEE doubles without FMA contraction and ``math.exp`` /
``math.sqrt`` are the C library's, so the arithmetic follows the reference's
operation order bit for bit (checked by tests/test_setup.py).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field as dfield
from typing import Callable, Optional

import numpy as np

from . import abi
from .scene import DensityGrid, FlatScene, aperture, plane_mirror, sensor as make_sensor, \
    singlet as make_singlet, thin_lens

M64 = 0xFFFFFFFFFFFFFFFF
K_CALIBRATION_SOURCE = 0xCA1   # engine.cpp:25


# ----------------------------------------------------------------- core.hpp
def mix_bits(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class CounterRng:
    """core.hpp:92-107."""

    def __init__(self, seed: int, stream: int = 0, element: int = 0):
        self.key = mix_bits((mix_bits((mix_bits(seed & M64) + stream) & M64) + element) & M64)
        self.n = 0

    def uniform(self, a: float | None = None, b: float | None = None) -> float:
        self.n += 1
        x = mix_bits((self.key + 0x9E3779B97F4A7C15 * self.n) & M64)
        u = math.ldexp(float(x >> 11), -53)
        return u if a is None else a + (b - a) * u


# ------------------------------------------------------ FP64 vector helpers
def _add(a, b): return (a[0] + b[0], a[1] + b[1], a[2] + b[2])
def _sub(a, b): return (a[0] - b[0], a[1] - b[1], a[2] - b[2])
def _mul(a, s): return (a[0] * s, a[1] * s, a[2] * s)
def _div(a, s): return (a[0] / s, a[1] / s, a[2] / s)
def _neg(a): return (-a[0], -a[1], -a[2])
def _dot(a, b): return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]
def _norm(a): return math.sqrt(_dot(a, a))
def _normalized(a): return _div(a, _norm(a))


# --------------------------------------------- probe-ray optics (setup only)
# The same element semantics as the device chain (optics.cpp:15-158); used by
# build_scene for the autofocus / magnification / paraxial-EFL probes, which
# the reference also traces on the host (engine.cpp:63-75, 321-341, 354-368).
def _radial(p, ap, ax):
    rel = _sub(p, ap)
    return _norm(_sub(rel, _mul(ax, _dot(rel, ax))))


def _plane_cap(o, d, point, axis, clear):
    denom = _dot(d, axis)
    if denom == 0.0:
        return None
    t = _dot(_sub(point, o), axis) / denom
    if t <= 1e-12:
        return None
    p = _add(o, _mul(d, t))
    if _radial(p, point, axis) > clear:
        return None
    return p, (axis if denom < 0.0 else _neg(axis))


def _v(v): return (v.x, v.y, v.z)


def _sphere(o, d, s: abi.Surface):
    if not math.isfinite(s.curvature_radius):
        return _plane_cap(o, d, _v(s.vertex), _v(s.axis), s.aperture_radius)
    vertex, axis, R = _v(s.vertex), _v(s.axis), s.curvature_radius
    center = _add(vertex, _mul(axis, R))
    oc = _sub(o, center)
    b = _dot(oc, d)
    c = _dot(oc, oc) - R * R
    disc = b * b - c
    if disc < 0.0:
        return None
    sq = math.sqrt(disc)
    for t in (-b - sq, -b + sq):
        if t <= 1e-12:
            continue
        p = _add(o, _mul(d, t))
        if _dot(_sub(p, center), _sub(vertex, center)) <= 0.0:
            continue
        if _radial(p, vertex, axis) > s.aperture_radius:
            continue
        n = _div(_sub(p, center), abs(R))
        if _dot(d, n) > 0.0:
            n = _neg(n)
        return p, n
    return None


def _refract(d, n, ni, nf):
    eta = ni / nf
    cos_i = -_dot(d, n)
    k = 1.0 - eta * eta * (1.0 - cos_i * cos_i)
    if k < 0.0:
        return None
    return _normalized(_add(_mul(d, eta), _mul(n, eta * cos_i - math.sqrt(k))))


def propagate_chain(o, d, elements):
    """Returns (origin, dir, reason) with reason 0 = transmitted (optics.cpp:143-158)."""
    for e in elements:
        if e.kind == abi.RB_ELEM_APERTURE:
            c, nrm = _v(e.center), _v(e.axis)
            denom = _dot(d, nrm)
            if denom == 0.0:
                return o, d, 2
            t = _dot(_sub(c, o), nrm) / denom
            if t <= 1e-12:
                return o, d, 2
            if _norm(_sub(_add(o, _mul(d, t)), c)) > e.radius:
                return o, d, 1
        elif e.kind == abi.RB_ELEM_THIN_LENS:
            c, ax = _v(e.center), _v(e.axis)
            hit = _plane_cap(o, d, c, ax, 0.5 * e.diameter)
            if hit is None:
                return o, d, 2
            dz = _dot(d, ax)
            if dz <= 0.0:
                return o, d, 2
            fp = _add(c, _mul(d, e.focal_length / dz))
            o, d = hit[0], _normalized(_mul(_sub(fp, hit[0]), 1.0 if e.focal_length > 0.0 else -1.0))
        elif e.kind == abi.RB_ELEM_SINGLET:
            h1 = _sphere(o, d, e.front)
            if h1 is None:
                return o, d, 2
            d1 = _refract(d, h1[1], e.front.n_before, e.front.n_after)
            if d1 is None:
                return o, d, 3
            h2 = _sphere(h1[0], d1, e.back)
            if h2 is None:
                return h1[0], d1, 2
            d2 = _refract(d1, h2[1], e.back.n_before, e.back.n_after)
            if d2 is None:
                return h1[0], d1, 3
            o, d = h2[0], d2
        else:
            hit = _sphere(o, d, e.front)
            if hit is None:
                return o, d, 2
            o, d = hit[0], _sub(d, _mul(hit[1], 2.0 * _dot(d, hit[1])))
    return o, d, 0


def intersect_sensor(o, d, s: abi.Sensor):
    """sensor.cpp:27-34."""
    n, c = _v(s.normal), _v(s.center)
    denom = _dot(d, n)
    if denom == 0.0:
        return None
    t = _dot(_sub(c, o), n) / denom
    if t <= 0.0:
        return None
    p = _sub(_add(o, _mul(d, t)), c)
    return _dot(p, _v(s.e_u)), _dot(p, _v(s.e_v))


# ------------------------------------------------------------- config.hpp
@dataclass
class ExperimentConfig:
    source: dict = dfield(default_factory=dict)
    medium: dict = dfield(default_factory=dict)
    gladstone_dale: float = 2.26e-4
    ambient_rho: float = 1.225
    z_dot_to_volume: float = 0.25
    z_volume_to_lens: float = 0.73
    optics: list = dfield(default_factory=list)
    sensor: dict = dfield(default_factory=dict)
    bundle: dict = dfield(default_factory=dict)
    trace: dict = dfield(default_factory=dict)
    bos: dict = dfield(default_factory=dict)
    run: dict = dfield(default_factory=dict)
    # in-memory medium override (the reference's GVOL path, without a file)
    density: Optional[DensityGrid] = None


class ConfigError(RuntimeError):
    pass


def _fail(msg):
    raise ConfigError("config: " + msg)


def _auto(v, key):
    if isinstance(v, str):
        if v == "auto":
            return 0.0
        _fail(key + ': expected a number or "auto"')
    return float(v)


def parse_config(src) -> ExperimentConfig:
    """parse_config_json (config.cpp:109-196), defaults from config.hpp:15-116."""
    j = json.loads(src) if isinstance(src, str) else src
    c = ExperimentConfig()
    sc = j.get("scene", {})
    s = sc.get("source", {})
    st = s.get("type", "dots")
    if st == "dots":
        c.source = {"type": "dots", "extent": tuple(s.get("extent_m", (0.02, 0.02))),
                    "dots_per_region": float(s.get("density_per_32px_region", 20.0)),
                    "count": int(s.get("count", -1)), "dot_diameter": float(s.get("dot_diameter_m", 1e-4)),
                    "seed": int(s.get("seed", 1))}
    elif st == "particles":
        c.source = {"type": "particles", "count": int(s.get("count", 0)),
                    "diameter": float(s.get("diameter_m", 5e-6)), "seed": int(s.get("seed", 1)),
                    "box_lo": tuple(s.get("box_lo_m", (0.0, 0.0, 0.0))),
                    "box_hi": tuple(s.get("box_hi_m", (0.0, 0.0, 0.0)))}
    else:
        _fail(f"unknown source type '{st}'")
    m = sc.get("medium", {})
    mt = m.get("type", "none")
    if mt not in ("none", "gvol", "uniform_gradient_slab", "gaussian_blob_slab"):
        _fail(f"unknown medium type '{mt}'")
    nodes = m.get("nodes", (33, 33, 5))
    c.medium = {"type": mt, "path": m.get("path", ""), "rho0": float(m.get("rho0_kg_m3", 1.225)),
                "grad": tuple(m.get("grad_kg_m4", (0.0, 0.0))),
                "amplitude": float(m.get("amplitude_kg_m3", 0.5)), "sigma": float(m.get("sigma_m", 0.004)),
                "extent": tuple(m.get("extent_m", (0.032, 0.032))), "depth": float(m.get("depth_m", 0.01)),
                "nx": int(nodes[0]), "ny": int(nodes[1]), "nz": int(nodes[2])}
    c.gladstone_dale = float(sc.get("gladstone_dale_m3_kg", c.gladstone_dale))
    c.ambient_rho = float(sc.get("ambient_rho_kg_m3", c.ambient_rho))
    g = j.get("geometry", {})
    c.z_dot_to_volume = float(g.get("z_dot_to_volume_m", c.z_dot_to_volume))
    c.z_volume_to_lens = float(g.get("z_volume_to_lens_m", c.z_volume_to_lens))
    for e in j.get("optics", []):
        t = e.get("type", "")
        if t not in ("aperture", "thin_lens", "singlet", "mirror_plane"):
            _fail(f"unknown optics element type '{t}'")
        c.optics.append({"type": t, "f_number": float(e.get("f_number", 0.0)),
                         "radius": float(e.get("radius_m", 0.0)),
                         "focal_length": float(e.get("focal_length_m", 0.0)),
                         "diameter": float(e.get("diameter_m", 0.0)), "r1": float(e.get("r1_m", 0.0)),
                         "r2": float(e.get("r2_m", 0.0)), "thickness": float(e.get("thickness_m", 0.0)),
                         "glass_index": float(e.get("glass_index", 1.5)),
                         "z": float(e["z_m"]) if "z_m" in e else None})
    se = j.get("sensor", {})
    res = se.get("resolution", (256, 256))
    c.sensor = {"width": int(res[0]), "height": int(res[1]), "pitch": float(se.get("pitch_m", 10e-6)),
                "bit_depth": int(se.get("bit_depth", 16)), "gain": _auto(se.get("gain", 0.0), "sensor.gain"),
                "distance": _auto(se.get("distance_m", 0.0), "sensor.distance_m"),
                "window_sigmas": float(se.get("spot_window_sigmas", 4.0)),
                "pi_factor": bool(se.get("diffraction_pi_factor", True)),
                "f_number": float(se.get("f_number", 0.0))}
    b = j.get("bundle", {})
    sampling = b.get("sampling", "stratified")
    if sampling not in ("stratified", "uniform-random"):
        _fail("bundle.sampling must be 'stratified' or 'uniform-random'")
    c.bundle = {"rays": int(b.get("rays_per_source", 10000)),
                "sampling": abi.RB_SAMPLING_STRATIFIED if sampling == "stratified" else abi.RB_SAMPLING_UNIFORM,
                "seed": int(b.get("seed", 1234)), "wavelength": float(b.get("wavelength_m", 500e-9))}
    t = j.get("trace", {})
    c.trace = {"delta_xi": float(t.get("delta_xi_m", 0.0)), "max_steps": int(t.get("max_steps", 0))}
    bo = j.get("bos", {})
    c.bos = {"magnification": float(bo.get("magnification", 0.0))}
    c.run = dict(j.get("run", {}))
    validate(c)
    return c


def validate(c: ExperimentConfig):
    """ExperimentConfig::validate (config.cpp:206-247), hot-path relevant part."""
    s = c.source
    if s["type"] == "dots":
        if s["extent"][0] <= 0 or s["extent"][1] <= 0:
            _fail("source extent must be positive")
        if s["count"] < 0 and s["dots_per_region"] <= 0:
            _fail("source density must be positive")
    elif s["count"] <= 0:
        _fail("particle source needs a positive count")
    m = c.medium
    if m["type"] == "gvol" and c.density is None:
        if not m["path"]:
            _fail("gvol medium needs a path")
        if not os.path.exists(m["path"]):
            _fail("gvol file not found: " + m["path"])
    if m["type"] != "none":
        if m["depth"] <= 0.0:
            _fail("medium depth must be positive")
        if m["type"] != "gvol" and (m["nx"] < 2 or m["ny"] < 2 or m["nz"] < 2):
            _fail("medium grid must have at least 2 nodes per axis")
    if c.gladstone_dale <= 0.0:
        _fail("Gladstone-Dale constant must be positive")
    if c.ambient_rho < 0.0:
        _fail("ambient density must be >= 0")
    if c.z_dot_to_volume <= 0.0 or c.z_volume_to_lens <= 0.0:
        _fail("geometry distances must be positive")
    if not c.optics:
        _fail("optics chain must not be empty")
    for e in c.optics:
        if e["type"] == "thin_lens" and e["focal_length"] == 0.0:
            _fail("thin lens needs a focal length")
        if e["type"] == "singlet" and e["thickness"] <= 0.0:
            _fail("singlet needs a positive thickness")
        if e["type"] in ("thin_lens", "singlet") and e["diameter"] <= 0.0:
            _fail("lens needs a positive diameter")
        if e["type"] == "aperture" and e["radius"] <= 0.0 and e["f_number"] <= 0.0:
            _fail("aperture needs radius_m or f_number")
    se = c.sensor
    if se["width"] < 1 or se["height"] < 1:
        _fail("sensor resolution must be positive")
    if se["pitch"] <= 0.0:
        _fail("sensor pitch must be positive")
    if se["bit_depth"] not in (8, 10, 12, 16):
        _fail("sensor bit depth must be one of 8, 10, 12, 16")
    if c.bundle["rays"] < 1:
        _fail("rays_per_source must be >= 1")
    if c.bundle["wavelength"] <= 0.0:
        _fail("wavelength must be positive")


# ----------------------------------------------------------------- media
def load_gvol(path: str) -> DensityGrid:
    """load_density_volume (scene.cpp:212-240): 'GVOL1 nx ny nz dx dy dz ox oy oz' + LE float32."""
    with open(path, "rb") as f:
        header = f.readline().decode().split()
        if len(header) != 10 or header[0] != "GVOL1":
            raise RuntimeError("load_density_volume: malformed GVOL header in " + path)
        nx, ny, nz = (int(v) for v in header[1:4])
        sp = tuple(float(v) for v in header[4:7])
        org = tuple(float(v) for v in header[7:10])
        cnt = nx * ny * nz
        rho = np.frombuffer(f.read(cnt * 4), dtype="<f4")
        if rho.size != cnt:
            raise RuntimeError("load_density_volume: truncated data in " + path)
    return DensityGrid(nx, ny, nz, org, sp, rho.astype(np.float32))


def save_gvol(grid: DensityGrid, path: str):
    """save_density_volume (scene.cpp:242-255)."""
    with open(path, "wb") as f:
        f.write(("GVOL1 %d %d %d %.17g %.17g %.17g %.17g %.17g %.17g\n" % (
            grid.nx, grid.ny, grid.nz, *grid.spacing, *grid.origin)).encode())
        f.write(np.ascontiguousarray(grid.rho, dtype="<f4").tobytes())


def build_medium_volume(c: ExperimentConfig) -> DensityGrid:
    """engine.cpp:27-61 (+ stack_2d_slice, scene.cpp:35-51)."""
    m = c.medium
    zc = c.z_dot_to_volume
    if m["type"] == "gvol" or c.density is not None:
        g = c.density if c.density is not None else load_gvol(m["path"])
        lo, hi = g.bounds()
        center = (lo + hi) * 0.5
        shift = (0.0 - center[0], 0.0 - center[1], zc - center[2])
        return DensityGrid(g.nx, g.ny, g.nz, (g.origin[0] + shift[0], g.origin[1] + shift[1],
                                              g.origin[2] + shift[2]), g.spacing, g.rho,
                           c.gladstone_dale)
    nx, ny = m["nx"], m["ny"]
    dx = m["extent"][0] / (nx - 1)
    dy = m["extent"][1] / (ny - 1)
    ox, oy = -0.5 * m["extent"][0], -0.5 * m["extent"][1]
    sl = np.empty(nx * ny, dtype=np.float32)
    for j in range(ny):
        for i in range(nx):
            x = ox + i * dx
            y = oy + j * dy
            rho = m["rho0"]
            if m["type"] == "uniform_gradient_slab":
                rho += m["grad"][0] * x + m["grad"][1] * y
            elif m["type"] == "gaussian_blob_slab":
                rho += m["amplitude"] * math.exp(-(x * x + y * y) / (2.0 * m["sigma"] * m["sigma"]))
            sl[j * nx + i] = rho
    nz = m["nz"]
    dz = m["depth"] / (nz - 1)
    return DensityGrid(nx, ny, nz, (ox, oy, zc - 0.5 * m["depth"]), (dx, dy, dz),
                       np.tile(sl, nz), c.gladstone_dale)


# -------------------------------------------------------------- resolve
@dataclass
class SetupInfo:
    lens_plane_z: float = 0.0
    focal_length: float = 0.0
    f_number: float = 0.0
    magnification: float = 0.0
    gain: float = 1.0
    ambient_index: float = 1.0
    volume_center_z: float = 0.0
    depth: float = 0.0
    bit_depth: int = 16
    dot_positions: Optional[np.ndarray] = None


def diffraction_diameter(f_number, magnification, wavelength, pi_factor=True):
    """sensor.cpp:36-42."""
    base = 2.44 * f_number * (magnification + 1.0) * wavelength
    return math.pi * base if pi_factor else base


def _paraxial_efl(lens: abi.Element) -> float:
    """engine.cpp:63-75."""
    h = 1e-4
    o, d, r = propagate_chain((h, 0.0, lens.front.vertex.z - 0.01), (0.0, 0.0, 1.0), [lens])
    if r:
        raise RuntimeError("engine: paraxial probe blocked by lens")
    slope = d[0] / d[2]
    if slope == 0.0:
        raise RuntimeError("engine: lens is afocal at paraxial height")
    return -h / slope


def build_scene(c: ExperimentConfig,
                calibrate: Optional[Callable[[FlatScene], np.ndarray]] = None):
    """build_scene_setup (engine.cpp:228-427).  Returns (FlatScene, DensityGrid | None, SetupInfo).

    ``calibrate(scene)`` must return the FP64 image of one bundle from the
    calibration source (engine.cpp:396-412); pass ``None`` to require a
    configured gain.
    """
    validate(c)
    info = SetupInfo()
    info.ambient_index = c.gladstone_dale * c.ambient_rho + 1.0
    if c.ambient_rho < 0.0:
        raise ValueError("gladstone_dale: negative density")
    info.volume_center_z = c.z_dot_to_volume
    depth = c.medium["depth"]
    grid = None
    delta_xi, max_steps = 0.0, 100000   # StepParams defaults, grin.hpp:23-26
    if c.medium["type"] != "none" or c.density is not None:
        grid = build_medium_volume(c)
        depth = (grid.nz - 1) * grid.spacing[2]
        delta_xi = c.trace["delta_xi"] if c.trace["delta_xi"] > 0.0 else 0.5 * min(grid.spacing)
        if c.trace["max_steps"] > 0:
            max_steps = c.trace["max_steps"]
        else:
            lo, hi = grid.bounds()
            ext = (hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2])
            max_steps = int(4.0 * _norm(ext) / delta_xi) + 64
    z_lens = c.z_dot_to_volume + c.z_volume_to_lens
    info.lens_plane_z = z_lens
    axis = (0.0, 0.0, 1.0)
    efl, last_exit_z, ap_index = 0.0, z_lens, -1
    elements, element_z = [], []
    for k, ec in enumerate(c.optics):
        z = ec["z"] if ec["z"] is not None else z_lens
        element_z.append(z)
        if ec["type"] == "thin_lens":
            elements.append(thin_lens((0.0, 0.0, z), axis, ec["focal_length"], ec["diameter"]))
            if efl == 0.0:
                efl = ec["focal_length"]
            last_exit_z = max(last_exit_z, z)
        elif ec["type"] == "singlet":
            r1 = math.inf if ec["r1"] == 0.0 else ec["r1"]
            r2 = math.inf if ec["r2"] == 0.0 else ec["r2"]
            lens = make_singlet((0.0, 0.0, z), axis, r1, r2, ec["thickness"], ec["glass_index"],
                                ec["diameter"], info.ambient_index)
            if efl == 0.0:
                efl = _paraxial_efl(lens)
            elements.append(lens)
            last_exit_z = max(last_exit_z, z + ec["thickness"])
        elif ec["type"] == "aperture":
            if ap_index < 0:
                ap_index = k
            elements.append(aperture((0.0, 0.0, z), axis, ec["radius"]))
        else:
            elements.append(plane_mirror((0.0, 0.0, z), axis, ec["diameter"]))
    info.focal_length = efl
    if ap_index >= 0:
        radius = c.optics[ap_index]["radius"]
        if radius <= 0.0:
            if efl <= 0.0:
                raise RuntimeError("engine: aperture f_number needs a lens focal length")
            radius = efl / (2.0 * c.optics[ap_index]["f_number"])
        elements[ap_index].radius = radius
        pupil_center, pupil_radius = (0.0, 0.0, element_z[ap_index]), radius
    else:
        lens_z, lens_r = z_lens, 0.0
        for k, ec in enumerate(c.optics):
            if ec["type"] in ("thin_lens", "singlet"):
                lens_z, lens_r = element_z[k], 0.499 * ec["diameter"]
                break
        if lens_r <= 0.0:
            raise RuntimeError("engine: no aperture or lens to aim rays at")
        pupil_center, pupil_radius = (0.0, 0.0, lens_z), lens_r
    info.f_number = c.sensor["f_number"] if c.sensor["f_number"] > 0.0 else \
        (efl / (2.0 * pupil_radius) if efl > 0.0 else 0.0)
    if c.sensor["distance"] > 0.0:
        sensor_z = last_exit_z + c.sensor["distance"]
    else:
        h = 0.05 * pupil_radius
        probes = []
        for sign in (1.0, -1.0):
            o, d, r = propagate_chain((0.0, 0.0, 0.0), _normalized((sign * h, 0.0, pupil_center[2])),
                                      elements)
            if r:
                raise RuntimeError("engine: autofocus probe blocked")
            probes.append((o, d))
        (ao, ad), (bo, bd) = probes
        sa, sb = ad[0] / ad[2], bd[0] / bd[2]
        if abs(sa - sb) < 1e-15:
            raise RuntimeError("engine: autofocus rays are parallel")
        sensor_z = (bo[0] - ao[0] + sa * ao[2] - sb * bo[2]) / (sa - sb)
        if sensor_z <= last_exit_z:
            raise RuntimeError("engine: autofocus found no real image behind the optics")
    sen = make_sensor((0.0, 0.0, sensor_z), (0.0, 0.0, -1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                      c.sensor["width"], c.sensor["height"], c.sensor["pitch"],
                      c.sensor["window_sigmas"])
    if c.bos["magnification"] > 0.0:
        info.magnification = c.bos["magnification"]
    else:
        xt = 2e-4
        o, d, r = propagate_chain((xt, 0.0, 0.0), _normalized(_sub(pupil_center, (xt, 0.0, 0.0))),
                                  elements)
        if r:
            raise RuntimeError("engine: magnification probe blocked")
        uv = intersect_sensor(o, d, sen)
        if uv is None:
            raise RuntimeError("engine: magnification probe missed the sensor")
        info.magnification = abs(uv[0]) / xt
    d_tau = diffraction_diameter(info.f_number, info.magnification, c.bundle["wavelength"],
                                 c.sensor["pi_factor"]) if info.f_number > 0.0 else 0.0
    s = c.source
    if s["type"] == "dots":
        if s["count"] >= 0:
            count = s["count"]
        else:  # generate_dot_pattern, scene.cpp:141-160
            region = 32.0 * c.sensor["pitch"] / info.magnification
            density = s["dots_per_region"] / (region * region)
            count = int(round_half_away(density * s["extent"][0] * s["extent"][1]))
        dots = np.empty((count, 2))
        ex, ey = s["extent"]
        for i in range(count):  # generate_dot_pattern_count, scene.cpp:162-176 (stream 0xd07)
            r = CounterRng(s["seed"], 0xD07, i)
            dots[i, 0] = r.uniform(-0.5 * ex, 0.5 * ex)
            dots[i, 1] = r.uniform(-0.5 * ey, 0.5 * ey)
        info.dot_positions = dots
        sources = np.column_stack([dots, np.zeros(count)])
    else:
        n = s["count"]
        lo, hi = s["box_lo"], s["box_hi"]
        sources = np.empty((n, 3))
        for i in range(n):  # generate_particle_field, scene.cpp:178-191 (stream 0x9a7)
            r = CounterRng(s["seed"], 0x9A7, i)
            sources[i] = (r.uniform(lo[0], hi[0]), r.uniform(lo[1], hi[1]), r.uniform(lo[2], hi[2]))
    scene = FlatScene(sources=sources, pupil_center=pupil_center, pupil_axis=axis,
                      pupil_radius=pupil_radius, rays_per_source=c.bundle["rays"],
                      sampling=c.bundle["sampling"], seed=c.bundle["seed"],
                      wavelength=c.bundle["wavelength"], delta_xi=delta_xi, max_steps=max_steps,
                      elements=elements, sensor=sen, d_tau=d_tau)
    info.bit_depth = c.sensor["bit_depth"]
    info.depth = depth
    if c.sensor["gain"] > 0.0:
        info.gain = c.sensor["gain"]
    else:
        if calibrate is None:
            raise RuntimeError("build_scene: gain 'auto' needs a calibrate callback")
        cal = scene.subset([0])
        cal.sources = np.zeros((1, 3))
        cal.source_ids = np.array([K_CALIBRATION_SOURCE], dtype=np.int64)
        img = calibrate(cal)
        peak = float(np.max(img))
        full = float((1 << info.bit_depth) - 1)
        info.gain = 0.9 * full / peak if peak > 0.0 else 1.0
    return scene, grid, info


def round_half_away(x: float) -> float:
    """std::llround."""
    return math.floor(x + 0.5) if x >= 0 else math.ceil(x - 0.5)


def quantize(image: np.ndarray, bit_depth: int, gain: float) -> np.ndarray:
    """quantize (sensor.cpp:124-135): llround(gain * v) clamped to [0, 2^bits - 1]."""
    v = gain * np.asarray(image, dtype=np.float64)
    big = np.abs(v) >= 2.0 ** 52          # already integral
    fl = np.floor(np.where(big, 0.0, v))
    frac = np.where(big, 0.0, v) - fl     # exact for |v| < 2^52
    r = np.where(big, v, np.where(v >= 0, fl + (frac >= 0.5), -np.floor(-v + 0.0) - ((-v - np.floor(-v)) >= 0.5)))
    return np.clip(r, 0, (1 << bit_depth) - 1).astype(np.uint16)


def write_pgm16(path: str, image_u16: np.ndarray, comments=()):
    """write_pgm16 (image_io.cpp:11-27): P5, maxval 65535, big-endian samples."""
    h, w = image_u16.shape
    with open(path, "wb") as f:
        f.write(b"P5\n")
        for cm in comments:
            f.write(f"# {cm}\n".encode())
        f.write(f"{w} {h}\n65535\n".encode())
        f.write(np.ascontiguousarray(image_u16, dtype=">u2").tobytes())
