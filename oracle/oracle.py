"""TEST INFRASTRUCTURE ONLY — Python handles on the two CPU checkers.

* :class:`COracle`   — ``oracle/liboracle.so``, the plain-C restatement of the
  reference hot path (``raybos_oracle.c``).
* :class:`Reference` — ``oracle/_ref/libraybos_ref.so``, the unmodified
  reference library compiled from /root/reference/proj/src by
  ``oracle/Makefile``, behind ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  Neither library is ever used
by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from paper_1812_05902_b200 import abi
from paper_1812_05902_b200.scene import FlatScene, FieldNodes, DensityGrid, TraceResult, report_from

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libraybos_ref.so")


def _err():
    return C.create_string_buffer(1024)


def _alloc_out(n_src: int, w: int, h: int, image: bool):
    hit = np.zeros((n_src, 2), dtype=np.float64)
    landed = np.zeros(n_src, dtype=np.int64)
    img = np.zeros((h, w), dtype=np.float64) if image else None
    out = abi.TraceOut()
    out.hit_sum = abi.dptr(hit) if n_src else None
    out.landed = abi.i64ptr(landed) if n_src else None
    out.image = abi.dptr(img) if image else None
    return out, hit, landed, img


class COracle:
    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        dp = C.POINTER(C.c_double)
        lib.oracle_trace.argtypes = [C.POINTER(abi.Scene), C.POINTER(abi.FieldDesc), dp, dp, dp, dp,
                                     C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int32,
                                     C.POINTER(C.c_uint64), C.POINTER(abi.TraceOut), C.c_char_p,
                                     C.c_size_t]
        lib.oracle_trace_rays.argtypes = [C.POINTER(abi.Scene), C.POINTER(abi.FieldDesc), dp, dp,
                                          dp, dp, C.c_int, C.c_int64, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int32), dp, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32), dp, C.c_char_p, C.c_size_t]
        lib.oracle_field_from_density.argtypes = [C.POINTER(abi.FieldDesc), C.POINTER(C.c_float),
                                                  C.c_double, dp, dp, dp, dp]
        lib.oracle_field_from_density.restype = None
        self.lib = lib

    @staticmethod
    def _field_args(field: Optional[FieldNodes]):
        if field is None:
            return None, None, None, None, None
        return (C.byref(field.desc()), abi.dptr(field.n), abi.dptr(field.gx), abi.dptr(field.gy),
                abi.dptr(field.gz))

    def trace(self, scene: FlatScene, field: Optional[FieldNodes], with_field=True,
              accumulate_image=True, shard_of=None, shard_index=0, fixed_point=False):
        s, keep = scene.to_c()
        out, hit, landed, img = _alloc_out(scene.n_sources, scene.width, scene.height,
                                           accumulate_image and not fixed_point)
        fixed = None
        if accumulate_image and fixed_point:
            fixed = np.zeros((scene.height, scene.width), dtype=np.uint64)
        err = _err()
        rc = self.lib.oracle_trace(C.byref(s), *self._field_args(field), int(with_field),
                                   int(accumulate_image),
                                   abi.i32ptr(shard_of) if shard_of is not None else None,
                                   int(shard_index),
                                   abi.u64ptr(fixed) if fixed is not None else None,
                                   C.byref(out), err, 1024)
        if rc:
            raise (ValueError if rc == abi.RB_E_INVALID else RuntimeError)(err.value.decode())
        res = TraceResult(hit, landed, img if not fixed_point else None, report_from(out))
        res.fixed = fixed
        return res

    def trace_rays(self, scene: FlatScene, field: Optional[FieldNodes], src, ray, with_field=True):
        s, keep = scene.to_c()
        src = np.ascontiguousarray(src, dtype=np.int64)
        ray = np.ascontiguousarray(ray, dtype=np.int32)
        n = src.shape[0]
        uv = np.zeros((n, 2))
        status = np.zeros(n, dtype=np.int32)
        steps = np.zeros(n, dtype=np.int32)
        exit_state = np.zeros((n, 6))
        err = _err()
        rc = self.lib.oracle_trace_rays(C.byref(s), *self._field_args(field), int(with_field), n,
                                        abi.i64ptr(src), abi.i32ptr(ray), abi.dptr(uv),
                                        abi.i32ptr(status), abi.i32ptr(steps),
                                        abi.dptr(exit_state), err, 1024)
        if rc:
            raise (ValueError if rc == abi.RB_E_INVALID else RuntimeError)(err.value.decode())
        return uv, status, steps, exit_state

    def field_from_density(self, grid: DensityGrid) -> FieldNodes:
        cnt = grid.nx * grid.ny * grid.nz
        arrs = [np.zeros(cnt) for _ in range(4)]
        rho = np.ascontiguousarray(grid.rho, dtype=np.float32)
        self.lib.oracle_field_from_density(C.byref(grid.desc()), abi.fptr(rho),
                                           grid.gladstone_dale, *[abi.dptr(a) for a in arrs])
        return FieldNodes(grid.nx, grid.ny, grid.nz, tuple(grid.origin), tuple(grid.spacing), *arrs)


class RefInfo(C.Structure):
    _fields_ = [("lens_plane_z", C.c_double), ("focal_length", C.c_double),
                ("f_number", C.c_double), ("magnification", C.c_double), ("gain", C.c_double),
                ("ambient_index", C.c_double), ("volume_center_z", C.c_double),
                ("d_tau", C.c_double), ("bit_depth", C.c_int32), ("has_field", C.c_int32),
                ("config_hash", C.c_uint64)]


def reference_available() -> bool:
    return os.path.exists(REF_LIB)


class Reference:
    """One reference SceneSetup (built by the reference's own build_scene_setup)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_LIB):
                raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle ref` where "
                                   "/root/reference exists")
            lib = C.CDLL(REF_LIB)
            vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
            dp = C.POINTER(C.c_double)
            lib.refshim_create_json.argtypes = [cp, C.POINTER(vp), cp, sz]
            lib.refshim_create_builtin.argtypes = [cp, C.POINTER(vp), cp, sz]
            lib.refshim_destroy.argtypes = [vp]
            lib.refshim_destroy.restype = None
            lib.refshim_export_scene.argtypes = [vp, C.POINTER(abi.Scene)]
            lib.refshim_export_scene.restype = None
            lib.refshim_info_get.argtypes = [vp, C.POINTER(RefInfo)]
            lib.refshim_info_get.restype = None
            lib.refshim_field_desc.argtypes = [vp, C.POINTER(abi.FieldDesc)]
            lib.refshim_field_nodes.argtypes = [vp, dp, dp, dp, dp]
            lib.refshim_field_nodes.restype = None
            lib.refshim_set_field_density.argtypes = [vp, C.POINTER(abi.FieldDesc),
                                                      C.POINTER(C.c_float), C.c_double, cp, sz]
            lib.refshim_clear_field.argtypes = [vp]
            lib.refshim_clear_field.restype = None
            lib.refshim_set_step.argtypes = [vp, C.c_double, C.c_int32]
            lib.refshim_set_step.restype = None
            lib.refshim_set_sources.argtypes = [vp, C.POINTER(abi.Vec3), C.c_int64]
            lib.refshim_set_sources.restype = None
            lib.refshim_set_bundle.argtypes = [vp, C.c_int32, C.c_int32, C.c_uint64]
            lib.refshim_set_bundle.restype = None
            lib.refshim_set_flat.argtypes = [vp, C.POINTER(abi.Scene)]
            lib.refshim_set_flat.restype = None
            lib.refshim_run_trace.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(abi.TraceOut), cp, sz]
            lib.refshim_trace_rays.argtypes = [vp, C.c_int, C.c_int64, C.POINTER(C.c_int64),
                                               C.POINTER(C.c_int32), dp, C.POINTER(C.c_int32),
                                               C.POINTER(C.c_int32), dp, cp, sz]
            lib.refshim_trace_debug.argtypes = [vp, C.c_int64, C.c_int32, dp, C.c_int64]
            lib.refshim_trace_debug.restype = C.c_int64
            lib.refshim_quantize.argtypes = [dp, C.c_int64, C.c_int, C.c_double,
                                             C.POINTER(C.c_uint16), cp, sz]
            lib.refshim_bos_metrics.argtypes = [vp, dp, C.POINTER(C.c_int64), dp,
                                                C.POINTER(C.c_int64), dp, cp, sz]
            cls._lib = lib
        return cls._lib

    def __init__(self, json_text: str | None = None, builtin: str | None = None):
        lib = self.lib()
        h = C.c_void_p()
        err = _err()
        if builtin is not None:
            rc = lib.refshim_create_builtin(builtin.encode(), C.byref(h), err, 1024)
        else:
            rc = lib.refshim_create_json(json_text.encode(), C.byref(h), err, 1024)
        if rc:
            raise RuntimeError(err.value.decode())
        self.h = h

    def close(self):
        if self.h:
            self.lib().refshim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def scene(self) -> FlatScene:
        s = abi.Scene()
        self.lib().refshim_export_scene(self.h, C.byref(s))
        return FlatScene.from_c(s)

    def info(self) -> RefInfo:
        i = RefInfo()
        self.lib().refshim_info_get(self.h, C.byref(i))
        return i

    def field(self) -> Optional[FieldNodes]:
        d = abi.FieldDesc()
        if not self.lib().refshim_field_desc(self.h, C.byref(d)):
            return None
        cnt = d.nx * d.ny * d.nz
        arrs = [np.zeros(cnt) for _ in range(4)]
        self.lib().refshim_field_nodes(self.h, *[abi.dptr(a) for a in arrs])
        return FieldNodes(d.nx, d.ny, d.nz, (d.origin.x, d.origin.y, d.origin.z),
                          (d.spacing.x, d.spacing.y, d.spacing.z), *arrs)

    def set_field_density(self, grid: DensityGrid):
        err = _err()
        rho = np.ascontiguousarray(grid.rho, dtype=np.float32)
        if self.lib().refshim_set_field_density(self.h, C.byref(grid.desc()), abi.fptr(rho),
                                                grid.gladstone_dale, err, 1024):
            raise RuntimeError(err.value.decode())

    def clear_field(self):
        self.lib().refshim_clear_field(self.h)

    def set_flat(self, scene: FlatScene):
        s, keep = scene.to_c()
        self.lib().refshim_set_flat(self.h, C.byref(s))

    def set_sources(self, sources: np.ndarray):
        src = np.ascontiguousarray(sources, dtype=np.float64)
        self.lib().refshim_set_sources(self.h, src.ctypes.data_as(C.POINTER(abi.Vec3)),
                                       src.shape[0])

    def run_trace(self, with_field=True, accumulate_image=True, threads=0, deterministic=True):
        sc = self.scene()
        out, hit, landed, img = _alloc_out(sc.n_sources, sc.width, sc.height, accumulate_image)
        err = _err()
        rc = self.lib().refshim_run_trace(self.h, int(with_field), int(accumulate_image), threads,
                                          int(deterministic), C.byref(out), err, 1024)
        if rc:
            raise (ValueError if rc == abi.RB_E_INVALID else RuntimeError)(err.value.decode())
        return TraceResult(hit, landed, img, report_from(out))

    def trace_rays(self, src, ray, with_field=True):
        src = np.ascontiguousarray(src, dtype=np.int64)
        ray = np.ascontiguousarray(ray, dtype=np.int32)
        n = src.shape[0]
        uv = np.zeros((n, 2))
        status = np.zeros(n, dtype=np.int32)
        steps = np.zeros(n, dtype=np.int32)
        exit_state = np.full((n, 6), np.nan)
        err = _err()
        rc = self.lib().refshim_trace_rays(self.h, int(with_field), n, abi.i64ptr(src),
                                           abi.i32ptr(ray), abi.dptr(uv), abi.i32ptr(status),
                                           abi.i32ptr(steps), abi.dptr(exit_state), err, 1024)
        if rc:
            raise RuntimeError(err.value.decode())
        return uv, status, steps, exit_state

    def trace_debug(self, dot: int, ray: int, cap: int = 100000) -> np.ndarray:
        """The reference trace_debug records (xi, r, t) of one ray, shape (n, 7)."""
        rec = np.zeros((cap, 7))
        n = self.lib().refshim_trace_debug(self.h, dot, ray, abi.dptr(rec), cap)
        return rec[:min(n, cap)].copy()

    def bos_metrics(self, ref: TraceResult, grad: TraceResult):
        m = np.zeros(6)
        err = _err()
        rh = np.ascontiguousarray(ref.hit_sum)
        gh = np.ascontiguousarray(grad.hit_sum)
        rc = self.lib().refshim_bos_metrics(self.h, abi.dptr(rh), abi.i64ptr(ref.landed),
                                            abi.dptr(gh), abi.i64ptr(grad.landed), abi.dptr(m),
                                            err, 1024)
        if rc:
            raise RuntimeError(err.value.decode())
        return {"rms_error": m[0], "peak_abs_error": m[1], "pearson": m[2], "peak_theory": m[3],
                "peak_measured": m[4], "nodes": int(m[5])}

    @classmethod
    def quantize(cls, image: np.ndarray, bit_depth: int, gain: float) -> np.ndarray:
        img = np.ascontiguousarray(image, dtype=np.float64).ravel()
        out = np.zeros(img.size, dtype=np.uint16)
        err = _err()
        if cls.lib().refshim_quantize(abi.dptr(img), img.size, bit_depth, gain,
                                      out.ctypes.data_as(C.POINTER(C.c_uint16)), err, 1024):
            raise RuntimeError(err.value.decode())
        return out.reshape(image.shape)
