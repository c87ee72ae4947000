"""The C-ABI library (include/raybos_gpu.h): loads without a GPU, exports every
declared symbol, and its ctypes mirror matches the C struct layout."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1812_05902_b200 import abi
from paper_1812_05902_b200.scene import FlatScene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "raybos_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*[\w\s\*]*?\b(rb_\w+)\s*\(", text, flags=re.M)))


def test_library_is_built_in_tree_and_loads_without_gpu():
    assert os.path.exists(abi.LIB_PATH), "run __graft_entry__.build() first"
    lib = abi.load_library()
    assert lib.rb_abi_version() == abi.RB_ABI_VERSION


def test_every_declared_symbol_is_exported():
    decl = declared_functions()
    assert len(decl) >= 14
    assert sorted(abi.EXPORTED_SYMBOLS) == decl
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (rb_\w+)", out))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_library_contains_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_ctypes_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    fields = {
        "rb_vec3": ["x", "y", "z"],
        "rb_surface": ["vertex", "axis", "curvature_radius", "aperture_radius", "n_before", "n_after"],
        "rb_element": ["kind", "center", "axis", "radius", "focal_length", "diameter", "front", "back"],
        "rb_sensor": ["center", "normal", "e_u", "e_v", "width_px", "height_px", "pitch", "window_sigmas"],
        "rb_scene": ["sources", "n_sources", "source_ids", "pupil_center", "pupil_axis",
                     "pupil_radius", "rays_per_source", "sampling", "seed", "wavelength",
                     "delta_xi", "max_steps", "n_elements", "elements", "sensor", "d_tau",
                     "config_hash"],
        "rb_field_desc": ["nx", "ny", "nz", "origin", "spacing"],
        "rb_trace_out": ["hit_sum", "landed", "image", "emitted", "landed_total", "lost",
                         "blocked_aperture", "blocked_miss", "blocked_tir", "blocked_sensor_miss",
                         "wall_seconds", "threads", "config_hash", "total_steps", "kernel_ms",
                         "quantized", "gain", "bit_depth", "kernel_launches", "image_fixed"],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "raybos_gpu.h"', 'int main(void){']
    for st, fs in fields.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                  check=True).stdout.splitlines())
    py = {"rb_vec3": abi.Vec3, "rb_surface": abi.Surface, "rb_element": abi.Element,
          "rb_sensor": abi.Sensor, "rb_scene": abi.Scene, "rb_field_desc": abi.FieldDesc,
          "rb_trace_out": abi.TraceOut}
    for st, cls in py.items():
        assert int(got[st]) == C.sizeof(cls), st
        for f in fields[st]:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, f"{st}.{f}"


def test_create_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = abi.load_library()
    ctx = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib.rb_create(1, 0, C.byref(ctx), err, 512)
    assert rc == abi.RB_E_NODEVICE
    assert b"no CPU fallback" in err.value


def _scene(n=1000, seed=0):
    rng = np.random.default_rng(seed)
    from paper_1812_05902_b200.scene import sensor
    return FlatScene(sources=np.column_stack([rng.uniform(-0.05, 0.05, (n, 2)), np.zeros(n)]),
                     pupil_center=(0, 0, 0.98), pupil_axis=(0, 0, 1.0), pupil_radius=0.004,
                     rays_per_source=100, sampling=0, seed=1, wavelength=5e-7, delta_xi=0.0,
                     max_steps=0, elements=[],
                     sensor=sensor((0, 0, 1.1), (0, 0, -1), (1, 0, 0), (0, 1, 0), 64, 64, 1e-5),
                     d_tau=4.7e-5)


@pytest.mark.parametrize("count", [1, 2, 3, 8])
def test_plan_shards_partitions_sources(count):
    from paper_1812_05902_b200.engine import plan_shards
    sc = _scene(1000)
    plan = plan_shards(sc, count)
    assert plan.shape == (1000,) and plan.min() >= 0 and plan.max() < count
    sizes = np.bincount(plan, minlength=count)
    assert sizes.max() - sizes.min() <= 32          # dealt in tiles of 32
    assert np.array_equal(plan, plan_shards(sc, count))  # deterministic


def test_plan_shards_tiles_are_spatially_compact():
    """Sources of one shard tile are neighbours (Z-order), so a tile's cones share grid cells."""
    from paper_1812_05902_b200.engine import plan_shards
    sc = _scene(4096, seed=3)
    plan = plan_shards(sc, 128)          # 128 shards x 32 sources: one tile per shard
    spread = []
    for k in range(128):
        p = sc.sources[plan == k, :2]
        spread.append(np.ptp(p, axis=0).max())
    # a random 32-subset spans ~the whole 0.1 m field; Z-order tiles are far smaller
    assert np.median(spread) < 0.03
