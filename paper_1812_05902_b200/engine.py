"""Python handle on the C-ABI: the reference's ``run_trace`` (engine.hpp:73-78)
on B200, plus the multi-process shard entry points.

Everything here is a thin ctypes call into ``libraybos_gpu.so``; the hot path
never runs in Python and there is no CPU fallback (constructing a
:class:`GpuTracer` without a B200 raises).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Union

import numpy as np

from . import abi
from .scene import DensityGrid, FieldNodes, FlatScene, TraceResult, report_from


class RaybosError(RuntimeError):
    pass


def _raise(lib, ctx, rc, what):
    msg = lib.rb_last_error(ctx).decode() if ctx else what
    if rc == abi.RB_E_INVALID:
        raise ValueError(msg)
    raise RaybosError(f"{what}: {msg}")


def plan_shards(scene: FlatScene, shard_count: int) -> np.ndarray:
    """rb_plan_shards: shard of every source (host only, no device needed)."""
    lib = abi.load_library()
    s, keep = scene.to_c()
    out = np.zeros(max(scene.n_sources, 1), dtype=np.int32)
    rc = lib.rb_plan_shards(C.byref(s), int(shard_count), abi.i32ptr(out))
    if rc:
        raise ValueError("rb_plan_shards failed")
    return out[: scene.n_sources]


def nccl_unique_id() -> bytes:
    """rb_nccl_unique_id: rank 0's communicator id, to hand to every rank."""
    lib = abi.load_library()
    buf = C.create_string_buffer(abi.RB_NCCL_UNIQUE_ID_BYTES)
    err = C.create_string_buffer(1024)
    rc = lib.rb_nccl_unique_id(buf, abi.RB_NCCL_UNIQUE_ID_BYTES, err, 1024)
    if rc:
        raise RaybosError(f"rb_nccl_unique_id failed: {err.value.decode()}")
    return buf.raw


class GpuTracer:
    """Owns an ``rb_ctx``: device streams, the resident density grid, buffers.

    ``GpuTracer(n)`` renders on devices first_device .. first_device+n-1 from
    this process (``devices=[...]`` names them explicitly);
    ``GpuTracer.for_rank(device, rank, world, uid)`` is one rank of a
    one-process-per-GPU job (rb_create_rank)."""

    def __init__(self, n_devices: int = 1, first_device: int = 0, devices=None, _ctx=None):
        self.lib = abi.load_library()
        self.ctx = C.c_void_p()
        err = C.create_string_buffer(1024)
        if _ctx is not None:
            self.ctx = _ctx
            return
        if devices is not None:
            arr = (C.c_int * len(devices))(*[int(d) for d in devices])
            rc = self.lib.rb_create_devices(arr, len(devices), C.byref(self.ctx), err, 1024)
        else:
            rc = self.lib.rb_create(int(n_devices), int(first_device), C.byref(self.ctx), err, 1024)
        if rc:
            raise RaybosError(f"rb_create failed: {err.value.decode()}")

    @classmethod
    def for_rank(cls, device: int, rank: int, world: int, uid: bytes | None) -> "GpuTracer":
        lib = abi.load_library()
        ctx = C.c_void_p()
        err = C.create_string_buffer(1024)
        idbuf = C.create_string_buffer(uid, abi.RB_NCCL_UNIQUE_ID_BYTES) if uid else None
        rc = lib.rb_create_rank(int(device), int(rank), int(world), idbuf,
                                abi.RB_NCCL_UNIQUE_ID_BYTES if uid else 0, C.byref(ctx), err, 1024)
        if rc:
            raise RaybosError(f"rb_create_rank failed: {err.value.decode()}")
        return cls(_ctx=ctx)

    def comm_info(self) -> dict:
        """rank / world / ranks of the NCCL communicator / NCCL version (0: stand-in)."""
        v = [C.c_int() for _ in range(4)]
        self.lib.rb_comm_info(self.ctx, *[C.byref(x) for x in v])
        return dict(zip(("rank", "world", "comm_ranks", "nccl_version"), (x.value for x in v)))

    def close(self):
        if self.ctx:
            self.lib.rb_destroy(self.ctx)
            self.ctx = C.c_void_p()
        for p in getattr(self, "_pinned", []):
            self.lib.rb_host_free(p)
        self._pinned = []

    def pinned(self, shape, dtype=np.float64) -> np.ndarray:
        """A numpy array in page-locked host memory (rb_host_alloc), owned by
        this tracer (freed by close): pass it as run_trace's image_out so the
        image comes back at full copy bandwidth."""
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = self.lib.rb_host_alloc(n)
        if not p:
            raise RaybosError("rb_host_alloc failed")
        if not hasattr(self, "_pinned"):
            self._pinned = []
        self._pinned.append(p)
        buf = (C.c_char * n).from_address(p)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def reset_plan(self):
        """rb_plan_reset: the next run_trace re-plans and re-uploads the sources."""
        self.lib.rb_plan_reset(self.ctx)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def n_devices(self) -> int:
        return self.lib.rb_device_count(self.ctx)

    # ---- field -------------------------------------------------------------
    def set_field(self, field: Union[FieldNodes, DensityGrid, None]):
        if field is None:
            self.lib.rb_clear_field(self.ctx)
            return
        d = field.desc()
        if isinstance(field, FieldNodes):
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                    (field.n, field.gx, field.gy, field.gz)]
            rc = self.lib.rb_set_field_nodes(self.ctx, C.byref(d), *[abi.dptr(a) for a in arrs])
        else:
            rho = np.ascontiguousarray(field.rho, dtype=np.float32)
            rc = self.lib.rb_set_field_density(self.ctx, C.byref(d), abi.fptr(rho),
                                               float(field.gladstone_dale))
        if rc:
            _raise(self.lib, self.ctx, rc, "set_field")

    def set_field_gvol(self, path: str, gladstone_dale: float = 2.26e-4,
                       z_center: Optional[float] = None, slab_bytes: int = 0) -> abi.FieldDesc:
        """rb_set_field_gvol: stream a GVOL file to the devices (host memory stays
        at two z-slabs) and build the grid there; returns the grid geometry."""
        d = abi.FieldDesc()
        zc = C.c_double(z_center) if z_center is not None else None
        rc = self.lib.rb_set_field_gvol(self.ctx, os.fsencode(path),
                                        C.byref(zc) if zc is not None else None,
                                        float(gladstone_dale), int(slab_bytes), C.byref(d))
        if rc:
            _raise(self.lib, self.ctx, rc, "set_field_gvol")
        return d

    def field_bytes(self) -> int:
        return int(self.lib.rb_field_bytes(self.ctx))

    # ---- run_trace -----------------------------------------------------------
    def run_trace(self, scene: FlatScene, with_field: bool = True, accumulate_image: bool = True,
                  image_out: Optional[np.ndarray] = None, quantize=None,
                  image_fixed_ptr: int = 0, host_image: bool = True) -> TraceResult:
        """rb_trace.  quantize=(bit_depth, gain) also returns the render tail's
        quantized uint16 image (computed on device) as result.quantized.
        image_fixed_ptr: a device buffer of W*H uint64 that receives the reduced
        fixed-point image (rb_trace_out.image_fixed); host_image=False then skips
        the FP64 host image.  In rank mode only rank 0 receives an image."""
        s, keep = scene.to_c()
        n = scene.n_sources
        hit = np.zeros((n, 2))
        landed = np.zeros(n, dtype=np.int64)
        img = None
        if accumulate_image and host_image:
            img = image_out if image_out is not None else np.empty((scene.height, scene.width))
            assert img.dtype == np.float64 and img.flags.c_contiguous and img.size == scene.width * scene.height
        out = abi.TraceOut()
        out.hit_sum = abi.dptr(hit) if n else None
        out.landed = abi.i64ptr(landed) if n else None
        out.image = abi.dptr(img) if img is not None else None
        out.image_fixed = int(image_fixed_ptr) if image_fixed_ptr else None
        qimg = None
        if quantize is not None and accumulate_image:
            qimg = np.zeros((scene.height, scene.width), dtype=np.uint16)
            out.quantized = qimg.ctypes.data_as(C.POINTER(C.c_uint16))
            out.bit_depth, out.gain = int(quantize[0]), float(quantize[1])
        rc = self.lib.rb_trace(self.ctx, C.byref(s), int(with_field), int(accumulate_image),
                               C.byref(out))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace")
        res = TraceResult(hit, landed, img, report_from(out))
        res.quantized = qimg
        return res

    def trace_bos_pair(self, scene: FlatScene):
        """rb_trace_bos_pair: bos_run's reference and gradient traces in one pass.
        Returns (reference TraceResult, gradient TraceResult), stats only."""
        s, keep = scene.to_c()
        n = scene.n_sources
        res = []
        outs = []
        for _ in range(2):
            hit = np.zeros((n, 2))
            landed = np.zeros(n, dtype=np.int64)
            o = abi.TraceOut()
            o.hit_sum = abi.dptr(hit) if n else None
            o.landed = abi.i64ptr(landed) if n else None
            res.append((hit, landed))
            outs.append(o)
        rc = self.lib.rb_trace_bos_pair(self.ctx, C.byref(s), C.byref(outs[0]), C.byref(outs[1]))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace_bos_pair")
        return tuple(TraceResult(h, l, None, report_from(o)) for (h, l), o in zip(res, outs))

    def trace_debug(self, scene: FlatScene, source_index: int, ray_index: int,
                    max_records: int = 100000) -> np.ndarray:
        """rb_trace_debug: StepObserver records (xi, r, t) of one ray, shape (n, 7)."""
        s, keep = scene.to_c()
        rec = np.zeros((max_records, 7))
        n = C.c_int64()
        rc = self.lib.rb_trace_debug(self.ctx, C.byref(s), int(source_index), int(ray_index),
                                     abi.dptr(rec), max_records, C.byref(n))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace_debug")
        return rec[:min(n.value, max_records)].copy()

    def trace_shard(self, scene: FlatScene, with_field: bool, accumulate_image: bool,
                    shard_index: int, shard_count: int, image_fixed_ptr: int,
                    hit: Optional[np.ndarray] = None, landed: Optional[np.ndarray] = None) -> dict:
        """rb_trace_shard; image_fixed_ptr is a device pointer to W*H uint64."""
        s, keep = scene.to_c()
        n = scene.n_sources
        hit = hit if hit is not None else np.zeros((n, 2))
        landed = landed if landed is not None else np.zeros(n, dtype=np.int64)
        out = abi.TraceOut()
        out.hit_sum = abi.dptr(hit) if n else None
        out.landed = abi.i64ptr(landed) if n else None
        rc = self.lib.rb_trace_shard(self.ctx, C.byref(s), int(with_field), int(accumulate_image),
                                     int(shard_index), int(shard_count),
                                     C.c_void_p(int(image_fixed_ptr)) if image_fixed_ptr else None,
                                     C.byref(out))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace_shard")
        rep = report_from(out)
        rep["hit_sum"] = hit
        rep["landed_per_source"] = landed
        return rep

    def image_from_fixed(self, image_fixed_ptr: int, shape) -> np.ndarray:
        img = np.empty(shape, dtype=np.float64)
        rc = self.lib.rb_image_from_fixed(self.ctx, C.c_void_p(int(image_fixed_ptr)), img.size,
                                          abi.dptr(img))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_image_from_fixed")
        return img

    def trace_rays_fp64(self, scene: FlatScene, src, ray, with_field: bool = True):
        """FP64 validation build of the per-ray replay (rb_trace_rays_fp64)."""
        return self.trace_rays(scene, src, ray, with_field, fp64=True)

    def trace_stats_fp64(self, scene: FlatScene, with_field: bool = True) -> TraceResult:
        """FP64 validation build of the per-source DotHitStats (rb_trace_stats_fp64)."""
        s, keep = scene.to_c()
        n = scene.n_sources
        hit = np.zeros((n, 2))
        landed = np.zeros(n, dtype=np.int64)
        out = abi.TraceOut()
        out.hit_sum = abi.dptr(hit) if n else None
        out.landed = abi.i64ptr(landed) if n else None
        rc = self.lib.rb_trace_stats_fp64(self.ctx, C.byref(s), int(with_field), C.byref(out))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace_stats_fp64")
        return TraceResult(hit, landed, None, report_from(out))

    def trace_rays(self, scene: FlatScene, src, ray, with_field: bool = True, fp64: bool = False):
        s, keep = scene.to_c()
        src = np.ascontiguousarray(src, dtype=np.int64)
        ray = np.ascontiguousarray(ray, dtype=np.int32)
        n = src.shape[0]
        uv = np.zeros((n, 2))
        status = np.zeros(n, dtype=np.int32)
        steps = np.zeros(n, dtype=np.int32)
        fn = self.lib.rb_trace_rays_fp64 if fp64 else self.lib.rb_trace_rays
        rc = fn(self.ctx, C.byref(s), int(with_field), n, abi.i64ptr(src),
                                    abi.i32ptr(ray), abi.dptr(uv), abi.i32ptr(status),
                                    abi.i32ptr(steps))
        if rc:
            _raise(self.lib, self.ctx, rc, "rb_trace_rays")
        return uv, status, steps
