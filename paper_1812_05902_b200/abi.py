"""ctypes mirror of include/raybos_gpu.h (the C-ABI drop-in boundary).

The product library ``libraybos_gpu.so`` is loaded from this package directory
and nowhere else; if it is missing the import of :func:`load_library` fails
loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

RB_ABI_VERSION = 2
RB_OK, RB_E_INVALID, RB_E_RUNTIME, RB_E_CUDA, RB_E_NODEVICE = 0, 1, 2, 3, 4
RB_RAY_LANDED, RB_RAY_LOST, RB_RAY_APERTURE, RB_RAY_MISSED, RB_RAY_TIR, RB_RAY_SENSOR_MISS = range(6)
RB_ELEM_APERTURE, RB_ELEM_SINGLET, RB_ELEM_THIN_LENS, RB_ELEM_MIRROR = range(4)
RB_SAMPLING_STRATIFIED, RB_SAMPLING_UNIFORM = 0, 1
RB_IMAGE_FIXED_SCALE = 2147483648.0


class Vec3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class Surface(C.Structure):
    _fields_ = [("vertex", Vec3), ("axis", Vec3), ("curvature_radius", C.c_double),
                ("aperture_radius", C.c_double), ("n_before", C.c_double),
                ("n_after", C.c_double)]


class Element(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("center", Vec3), ("axis", Vec3),
                ("radius", C.c_double), ("focal_length", C.c_double), ("diameter", C.c_double),
                ("front", Surface), ("back", Surface)]


class Sensor(C.Structure):
    _fields_ = [("center", Vec3), ("normal", Vec3), ("e_u", Vec3), ("e_v", Vec3),
                ("width_px", C.c_int32), ("height_px", C.c_int32), ("pitch", C.c_double),
                ("window_sigmas", C.c_double)]


class Scene(C.Structure):
    _fields_ = [("sources", C.POINTER(Vec3)), ("n_sources", C.c_int64),
                ("source_ids", C.POINTER(C.c_int64)),
                ("pupil_center", Vec3), ("pupil_axis", Vec3), ("pupil_radius", C.c_double),
                ("rays_per_source", C.c_int32), ("sampling", C.c_int32), ("seed", C.c_uint64),
                ("wavelength", C.c_double), ("delta_xi", C.c_double), ("max_steps", C.c_int32),
                ("n_elements", C.c_int32), ("elements", C.POINTER(Element)), ("sensor", Sensor),
                ("d_tau", C.c_double), ("config_hash", C.c_uint64)]


class FieldDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("reserved", C.c_int32),
                ("origin", Vec3), ("spacing", Vec3)]


class TraceOut(C.Structure):
    _fields_ = [("hit_sum", C.POINTER(C.c_double)), ("landed", C.POINTER(C.c_int64)),
                ("image", C.POINTER(C.c_double)),
                ("emitted", C.c_int64), ("landed_total", C.c_int64), ("lost", C.c_int64),
                ("blocked_aperture", C.c_int64), ("blocked_miss", C.c_int64),
                ("blocked_tir", C.c_int64), ("blocked_sensor_miss", C.c_int64),
                ("wall_seconds", C.c_double), ("threads", C.c_int32), ("k1_kernel", C.c_int32),
                ("config_hash", C.c_uint64), ("total_steps", C.c_int64),
                ("kernel_ms", C.c_double), ("quantized", C.POINTER(C.c_uint16)),
                ("gain", C.c_double), ("bit_depth", C.c_int32), ("kernel_launches", C.c_int32),
                ("image_fixed", C.c_void_p)]


def vec3(v) -> Vec3:
    return Vec3(float(v[0]), float(v[1]), float(v[2]))


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def i32ptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libraybos_gpu.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

# Every symbol include/raybos_gpu.h declares (checked by tests/test_capi.py).
EXPORTED_SYMBOLS = (
    "rb_create", "rb_destroy", "rb_last_error", "rb_abi_version", "rb_device_count",
    "rb_set_field_nodes", "rb_set_field_density", "rb_clear_field", "rb_field_bytes",
    "rb_trace", "rb_plan_shards", "rb_trace_shard", "rb_image_from_fixed", "rb_trace_rays",
    "rb_trace_rays_fp64", "rb_trace_stats_fp64", "rb_trace_debug", "rb_trace_bos_pair",
    "rb_set_field_gvol", "rb_create_devices", "rb_nccl_unique_id", "rb_create_rank",
    "rb_comm_info", "rb_plan_reset", "rb_host_alloc", "rb_host_free",
)
RB_NCCL_UNIQUE_ID_BYTES = 128

_lib = None


def load_library(path: str | None = None) -> C.CDLL:
    """Loads the in-tree CUDA library.  Raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("RAYBOS_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} is missing: the CUDA extension must be built (python -c "
            "'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(p)
    ctx_pp = C.POINTER(C.c_void_p)
    lib.rb_create.argtypes = [C.c_int, C.c_int, ctx_pp, C.c_char_p, C.c_size_t]
    lib.rb_create.restype = C.c_int
    lib.rb_create_devices.argtypes = [C.POINTER(C.c_int), C.c_int, ctx_pp, C.c_char_p, C.c_size_t]
    lib.rb_create_devices.restype = C.c_int
    lib.rb_nccl_unique_id.argtypes = [C.c_void_p, C.c_size_t, C.c_char_p, C.c_size_t]
    lib.rb_nccl_unique_id.restype = C.c_int
    lib.rb_create_rank.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t, ctx_pp,
                                   C.c_char_p, C.c_size_t]
    lib.rb_create_rank.restype = C.c_int
    lib.rb_comm_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4
    lib.rb_comm_info.restype = C.c_int
    lib.rb_plan_reset.argtypes = [C.c_void_p]
    lib.rb_plan_reset.restype = C.c_int
    lib.rb_host_alloc.argtypes = [C.c_size_t]
    lib.rb_host_alloc.restype = C.c_void_p
    lib.rb_host_free.argtypes = [C.c_void_p]
    lib.rb_host_free.restype = None
    lib.rb_destroy.argtypes = [C.c_void_p]
    lib.rb_destroy.restype = None
    lib.rb_last_error.argtypes = [C.c_void_p]
    lib.rb_last_error.restype = C.c_char_p
    lib.rb_abi_version.argtypes = []
    lib.rb_abi_version.restype = C.c_int
    lib.rb_device_count.argtypes = [C.c_void_p]
    lib.rb_device_count.restype = C.c_int
    lib.rb_set_field_nodes.argtypes = [C.c_void_p, C.POINTER(FieldDesc)] + [C.POINTER(C.c_double)] * 4
    lib.rb_set_field_nodes.restype = C.c_int
    lib.rb_set_field_density.argtypes = [C.c_void_p, C.POINTER(FieldDesc), C.POINTER(C.c_float),
                                         C.c_double]
    lib.rb_set_field_density.restype = C.c_int
    lib.rb_set_field_gvol.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double), C.c_double,
                                      C.c_int64, C.POINTER(FieldDesc)]
    lib.rb_set_field_gvol.restype = C.c_int
    lib.rb_clear_field.argtypes = [C.c_void_p]
    lib.rb_clear_field.restype = C.c_int
    lib.rb_field_bytes.argtypes = [C.c_void_p]
    lib.rb_field_bytes.restype = C.c_int64
    lib.rb_trace.argtypes = [C.c_void_p, C.POINTER(Scene), C.c_int, C.c_int, C.POINTER(TraceOut)]
    lib.rb_trace.restype = C.c_int
    lib.rb_plan_shards.argtypes = [C.POINTER(Scene), C.c_int64, C.POINTER(C.c_int32)]
    lib.rb_plan_shards.restype = C.c_int
    lib.rb_trace_shard.argtypes = [C.c_void_p, C.POINTER(Scene), C.c_int, C.c_int, C.c_int64,
                                   C.c_int64, C.c_void_p, C.POINTER(TraceOut)]
    lib.rb_trace_shard.restype = C.c_int
    lib.rb_image_from_fixed.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
    lib.rb_image_from_fixed.restype = C.c_int
    lib.rb_trace_rays.argtypes = [C.c_void_p, C.POINTER(Scene), C.c_int, C.c_int64,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]
    lib.rb_trace_rays.restype = C.c_int
    lib.rb_trace_rays_fp64.argtypes = lib.rb_trace_rays.argtypes
    lib.rb_trace_rays_fp64.restype = C.c_int
    lib.rb_trace_stats_fp64.argtypes = [C.c_void_p, C.POINTER(Scene), C.c_int, C.POINTER(TraceOut)]
    lib.rb_trace_stats_fp64.restype = C.c_int
    lib.rb_trace_debug.argtypes = [C.c_void_p, C.POINTER(Scene), C.c_int64, C.c_int32,
                                   C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int64)]
    lib.rb_trace_debug.restype = C.c_int
    lib.rb_trace_bos_pair.argtypes = [C.c_void_p, C.POINTER(Scene), C.POINTER(TraceOut),
                                      C.POINTER(TraceOut)]
    lib.rb_trace_bos_pair.restype = C.c_int
    if lib.rb_abi_version() != RB_ABI_VERSION:
        raise RuntimeError("libraybos_gpu.so ABI version mismatch; rebuild")
    if path is None:
        _lib = lib
    return lib
