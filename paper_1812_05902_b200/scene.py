"""Host-side scene containers for the C-ABI (include/raybos_gpu.h).

``FlatScene`` is the flattened form of the parts of ``raybos::SceneSetup``
(reference proj/include/raybos/engine.hpp:40-60) that ``run_trace`` reads;
``FieldNodes`` is ``GriddedField``'s node data (scene.hpp:68-105) and
``DensityGrid`` the ``DensityVolume`` it is built from (scene.hpp:25-40).
``TraceResult`` carries what ``TraceOutputs`` carries (engine.hpp:67-71).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field as dfield
from typing import Optional

import numpy as np

from . import abi


def _surf_to_dict(s: abi.Surface) -> dict:
    return {"vertex": [s.vertex.x, s.vertex.y, s.vertex.z], "axis": [s.axis.x, s.axis.y, s.axis.z],
            "curvature_radius": s.curvature_radius, "aperture_radius": s.aperture_radius,
            "n_before": s.n_before, "n_after": s.n_after}


def _surf_from_dict(d: dict) -> abi.Surface:
    return abi.Surface(abi.vec3(d["vertex"]), abi.vec3(d["axis"]), float(d["curvature_radius"]),
                       float(d["aperture_radius"]), float(d["n_before"]), float(d["n_after"]))


def element_to_dict(e: abi.Element) -> dict:
    return {"kind": e.kind, "center": [e.center.x, e.center.y, e.center.z],
            "axis": [e.axis.x, e.axis.y, e.axis.z], "radius": e.radius,
            "focal_length": e.focal_length, "diameter": e.diameter,
            "front": _surf_to_dict(e.front), "back": _surf_to_dict(e.back)}


def element_from_dict(d: dict) -> abi.Element:
    e = abi.Element()
    e.kind = int(d["kind"])
    e.center = abi.vec3(d["center"])
    e.axis = abi.vec3(d["axis"])
    e.radius = float(d["radius"])
    e.focal_length = float(d["focal_length"])
    e.diameter = float(d["diameter"])
    e.front = _surf_from_dict(d["front"])
    e.back = _surf_from_dict(d["back"])
    return e


def aperture(center, normal, radius) -> abi.Element:
    """raybos::Aperture (optics.hpp:80-84)."""
    e = abi.Element()
    e.kind = abi.RB_ELEM_APERTURE
    e.center, e.axis, e.radius = abi.vec3(center), abi.vec3(normal), float(radius)
    return e


def thin_lens(center, axis, focal_length, diameter) -> abi.Element:
    """raybos::ThinLensIdeal (optics.hpp:88-93)."""
    e = abi.Element()
    e.kind = abi.RB_ELEM_THIN_LENS
    e.center, e.axis = abi.vec3(center), abi.vec3(axis)
    e.focal_length, e.diameter = float(focal_length), float(diameter)
    return e


def singlet(front_vertex, axis, r1, r2, thickness, glass_index, diameter, ambient_index=1.0):
    """make_singlet (optics.cpp:69-83): two spherical caps on a common axis."""
    if thickness <= 0.0:
        raise ValueError("make_singlet: thickness must be positive")
    if diameter <= 0.0:
        raise ValueError("make_singlet: diameter must be positive")
    if glass_index <= 0.0:
        raise ValueError("make_singlet: glass index must be positive")
    fv = np.asarray(front_vertex, dtype=np.float64)
    ax = np.asarray(axis, dtype=np.float64)
    back_vertex = (fv[0] + ax[0] * thickness, fv[1] + ax[1] * thickness, fv[2] + ax[2] * thickness)
    e = abi.Element()
    e.kind = abi.RB_ELEM_SINGLET
    e.diameter = float(diameter)
    e.front = abi.Surface(abi.vec3(fv), abi.vec3(ax), float(r1), 0.5 * diameter,
                          float(ambient_index), float(glass_index))
    e.back = abi.Surface(abi.vec3(back_vertex), abi.vec3(ax), float(r2), 0.5 * diameter,
                         float(glass_index), float(ambient_index))
    return e


def plane_mirror(vertex, axis, diameter) -> abi.Element:
    e = abi.Element()
    e.kind = abi.RB_ELEM_MIRROR
    e.front = abi.Surface(abi.vec3(vertex), abi.vec3(axis), math.inf, 0.5 * diameter, 1.0, 1.0)
    return e


def rotation(axis, degrees) -> np.ndarray:
    """Right-handed rotation matrix about a unit axis (Rodrigues)."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    t = math.radians(degrees)
    K = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    return np.eye(3) + math.sin(t) * K + (1.0 - math.cos(t)) * (K @ K)


def sensor(center, normal, e_u, e_v, width_px, height_px, pitch, window_sigmas=4.0) -> abi.Sensor:
    """raybos::SensorModel (sensor.hpp:19-32) minus bit depth / gain."""
    return abi.Sensor(abi.vec3(center), abi.vec3(normal), abi.vec3(e_u), abi.vec3(e_v),
                      int(width_px), int(height_px), float(pitch), float(window_sigmas))


@dataclass
class FlatScene:
    sources: np.ndarray  # (n, 3) float64
    pupil_center: tuple
    pupil_axis: tuple
    pupil_radius: float
    rays_per_source: int
    sampling: int
    seed: int
    wavelength: float
    delta_xi: float
    max_steps: int
    elements: list
    sensor: abi.Sensor
    d_tau: float
    config_hash: int = 0
    source_ids: Optional[np.ndarray] = None

    @property
    def n_sources(self) -> int:
        return int(self.sources.shape[0])

    @property
    def width(self) -> int:
        return int(self.sensor.width_px)

    @property
    def height(self) -> int:
        return int(self.sensor.height_px)

    def to_c(self):
        """Returns (rb_scene, keepalive)."""
        src = np.ascontiguousarray(self.sources, dtype=np.float64).reshape(-1, 3)
        keep = [src]
        s = abi.Scene()
        s.sources = src.ctypes.data_as(C.POINTER(abi.Vec3)) if src.size else None
        s.n_sources = src.shape[0]
        if self.source_ids is not None:
            ids = np.ascontiguousarray(self.source_ids, dtype=np.int64)
            keep.append(ids)
            s.source_ids = ids.ctypes.data_as(C.POINTER(C.c_int64))
        s.pupil_center = abi.vec3(self.pupil_center)
        s.pupil_axis = abi.vec3(self.pupil_axis)
        s.pupil_radius = float(self.pupil_radius)
        s.rays_per_source = int(self.rays_per_source)
        s.sampling = int(self.sampling)
        s.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        s.wavelength = float(self.wavelength)
        s.delta_xi = float(self.delta_xi)
        s.max_steps = int(self.max_steps)
        arr = (abi.Element * max(1, len(self.elements)))(*self.elements)
        keep.append(arr)
        s.n_elements = len(self.elements)
        s.elements = C.cast(arr, C.POINTER(abi.Element))
        s.sensor = self.sensor
        s.d_tau = float(self.d_tau)
        s.config_hash = int(self.config_hash) & 0xFFFFFFFFFFFFFFFF
        return s, keep

    @staticmethod
    def from_c(s: abi.Scene) -> "FlatScene":
        n = int(s.n_sources)
        if n:
            buf = C.cast(s.sources, C.POINTER(C.c_double * (3 * n))).contents
            sources = np.frombuffer(buf, dtype=np.float64).reshape(n, 3).copy()
        else:
            sources = np.zeros((0, 3))
        ids = None
        if s.source_ids:
            ids = np.ctypeslib.as_array(s.source_ids, shape=(n,)).copy()
        elems = [abi.Element.from_buffer_copy(s.elements[i]) for i in range(s.n_elements)]
        return FlatScene(sources=sources, pupil_center=(s.pupil_center.x, s.pupil_center.y, s.pupil_center.z),
                         pupil_axis=(s.pupil_axis.x, s.pupil_axis.y, s.pupil_axis.z),
                         pupil_radius=s.pupil_radius, rays_per_source=s.rays_per_source,
                         sampling=s.sampling, seed=s.seed, wavelength=s.wavelength,
                         delta_xi=s.delta_xi, max_steps=s.max_steps, elements=elems,
                         sensor=abi.Sensor.from_buffer_copy(s.sensor), d_tau=s.d_tau,
                         config_hash=s.config_hash, source_ids=ids)

    def to_json(self) -> dict:
        se = self.sensor
        return {
            "sources": self.sources.tolist(),
            "source_ids": None if self.source_ids is None else self.source_ids.tolist(),
            "pupil_center": list(self.pupil_center), "pupil_axis": list(self.pupil_axis),
            "pupil_radius": self.pupil_radius, "rays_per_source": self.rays_per_source,
            "sampling": self.sampling, "seed": self.seed, "wavelength": self.wavelength,
            "delta_xi": self.delta_xi, "max_steps": self.max_steps,
            "elements": [element_to_dict(e) for e in self.elements],
            "sensor": {"center": [se.center.x, se.center.y, se.center.z],
                       "normal": [se.normal.x, se.normal.y, se.normal.z],
                       "e_u": [se.e_u.x, se.e_u.y, se.e_u.z], "e_v": [se.e_v.x, se.e_v.y, se.e_v.z],
                       "width_px": se.width_px, "height_px": se.height_px, "pitch": se.pitch,
                       "window_sigmas": se.window_sigmas},
            "d_tau": self.d_tau, "config_hash": self.config_hash,
        }

    @staticmethod
    def from_json(d: dict) -> "FlatScene":
        se = d["sensor"]
        return FlatScene(
            sources=np.asarray(d["sources"], dtype=np.float64).reshape(-1, 3),
            source_ids=None if d.get("source_ids") is None else np.asarray(d["source_ids"], dtype=np.int64),
            pupil_center=tuple(d["pupil_center"]), pupil_axis=tuple(d["pupil_axis"]),
            pupil_radius=d["pupil_radius"], rays_per_source=d["rays_per_source"],
            sampling=d["sampling"], seed=d["seed"], wavelength=d["wavelength"],
            delta_xi=d["delta_xi"], max_steps=d["max_steps"],
            elements=[element_from_dict(e) for e in d["elements"]],
            sensor=sensor(se["center"], se["normal"], se["e_u"], se["e_v"], se["width_px"],
                          se["height_px"], se["pitch"], se["window_sigmas"]),
            d_tau=d["d_tau"], config_hash=d["config_hash"])

    def dumps(self) -> str:
        return json.dumps(self.to_json())

    def with_camera_moved(self, rot, pivot) -> "FlatScene":
        """The same scene with the whole camera — pupil, every optical element
        (centres, axes, surface vertices / axes) and the sensor frame — turned
        by the rotation matrix ``rot`` about ``pivot``; sources unchanged.  The
        reference's SceneSetup carries general axes everywhere (optics.hpp:26-36,
        raygen.hpp:32-36, sensor.hpp:19-32) even though build_scene_setup only
        builds +z cameras (engine.cpp:258); this is how an off-axis perspective
        camera is expressed at the run_trace boundary."""
        R = np.asarray(rot, dtype=np.float64)
        c = np.asarray(pivot, dtype=np.float64)

        def pt(v):
            q = R @ (np.array([v.x, v.y, v.z]) - c) + c
            return abi.vec3(q)

        def ax(v):
            return abi.vec3(R @ np.array([v.x, v.y, v.z]))

        def surf(x: abi.Surface) -> abi.Surface:
            return abi.Surface(pt(x.vertex), ax(x.axis), x.curvature_radius, x.aperture_radius,
                               x.n_before, x.n_after)

        elems = []
        for e in self.elements:
            f = abi.Element.from_buffer_copy(e)
            f.center, f.axis = pt(e.center), ax(e.axis)
            f.front, f.back = surf(e.front), surf(e.back)
            elems.append(f)
        se = self.sensor
        out = FlatScene(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        pc = pt(abi.vec3(self.pupil_center))
        pa = ax(abi.vec3(self.pupil_axis))
        out.pupil_center = (pc.x, pc.y, pc.z)
        out.pupil_axis = (pa.x, pa.y, pa.z)
        out.elements = elems
        out.sensor = abi.Sensor(pt(se.center), ax(se.normal), ax(se.e_u), ax(se.e_v), se.width_px,
                                se.height_px, se.pitch, se.window_sigmas)
        return out

    def subset(self, idx) -> "FlatScene":
        """The same scene restricted to sources idx, keeping their RNG streams."""
        idx = np.asarray(idx, dtype=np.int64)
        base = self.source_ids if self.source_ids is not None else np.arange(self.n_sources)
        out = FlatScene(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        out.sources = self.sources[idx].copy()
        out.source_ids = np.asarray(base, dtype=np.int64)[idx].copy()
        return out


@dataclass
class FieldNodes:
    """GriddedField node data (scene.hpp:88-92): FP64 SoA, x-fastest."""
    nx: int
    ny: int
    nz: int
    origin: tuple
    spacing: tuple
    n: np.ndarray
    gx: np.ndarray
    gy: np.ndarray
    gz: np.ndarray

    def desc(self) -> abi.FieldDesc:
        return abi.FieldDesc(self.nx, self.ny, self.nz, 0, abi.vec3(self.origin),
                             abi.vec3(self.spacing))

    def bounds(self):
        lo = np.asarray(self.origin, dtype=np.float64)
        hi = lo + np.array([(self.nx - 1) * self.spacing[0], (self.ny - 1) * self.spacing[1],
                            (self.nz - 1) * self.spacing[2]])
        return lo, hi


@dataclass
class DensityGrid:
    """DensityVolume (scene.hpp:25-40): float rho, x-fastest, plus Gladstone-Dale K."""
    nx: int
    ny: int
    nz: int
    origin: tuple
    spacing: tuple
    rho: np.ndarray  # float32, size nx*ny*nz
    gladstone_dale: float = 2.26e-4

    def desc(self) -> abi.FieldDesc:
        return abi.FieldDesc(self.nx, self.ny, self.nz, 0, abi.vec3(self.origin),
                             abi.vec3(self.spacing))

    def bounds(self):
        lo = np.asarray(self.origin, dtype=np.float64)
        hi = lo + np.array([(self.nx - 1) * self.spacing[0], (self.ny - 1) * self.spacing[1],
                            (self.nz - 1) * self.spacing[2]])
        return lo, hi


@dataclass
class TraceResult:
    """TraceOutputs (engine.hpp:67-71) + RunReport (engine.hpp:19-36)."""
    hit_sum: np.ndarray            # (n, 2)
    landed: np.ndarray             # (n,)
    image: Optional[np.ndarray]    # (H, W) float64, row 0 = top
    report: dict = dfield(default_factory=dict)

    def accounting_ok(self) -> bool:
        r = self.report
        return r["emitted"] == r["landed"] + r["lost"] + r["blocked_aperture"] + \
            r["blocked_miss"] + r["blocked_tir"] + r["blocked_sensor_miss"]


def report_from(out: abi.TraceOut) -> dict:
    return {"emitted": out.emitted, "landed": out.landed_total, "lost": out.lost,
            "blocked_aperture": out.blocked_aperture, "blocked_miss": out.blocked_miss,
            "blocked_tir": out.blocked_tir, "blocked_sensor_miss": out.blocked_sensor_miss,
            "wall_seconds": out.wall_seconds, "threads": out.threads,
            "config_hash": out.config_hash, "total_steps": out.total_steps,
            "kernel_ms": out.kernel_ms, "kernel_launches": out.kernel_launches,
            "k1_kernel": out.k1_kernel}
