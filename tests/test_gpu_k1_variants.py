"""The two K1 work distributions — render_emitters (CTA-level chunks, the
default) and render_warps (warp-level items, RAYBOS_K1=warp) — must give the
same integers: the image, DotHitStats, counters and RK4 step totals, bit for bit."""
import numpy as np
import pytest

from golden_io import NAMES, load

pytestmark = pytest.mark.gpu
FIELD = [n for n in NAMES if load(n)[1] is not None]


CODE = {"cta": 1, "warp": 2}


def _run(tracer, scene, mode, monkeypatch):
    monkeypatch.setenv("RAYBOS_K1", mode)
    r = tracer.run_trace(scene, True, True)
    assert r.report["k1_kernel"] == CODE[mode]
    return r


@pytest.mark.parametrize("name", FIELD)
def test_warp_items_equal_cta_chunks(tracer, name, monkeypatch):
    scene, field, g = load(name)
    tracer.set_field(field)
    a = _run(tracer, scene, "cta", monkeypatch)
    b = _run(tracer, scene, "warp", monkeypatch)
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.hit_sum, b.hit_sum) and np.array_equal(a.landed, b.landed)
    for k in ("lost", "blocked_aperture", "blocked_miss", "blocked_tir", "blocked_sensor_miss",
              "total_steps"):
        assert a.report[k] == b.report[k], k


@pytest.mark.parametrize("name,scale", [("bos", 0.02), ("tomo", 0.003)])
def test_warp_items_equal_cta_chunks_on_bench_scenes(tracer, name, scale, monkeypatch):
    from paper_1812_05902_b200 import scenes
    scene, grid, info, desc = scenes.build(name, scale=scale)
    tracer.set_field(grid)
    a = _run(tracer, scene, "cta", monkeypatch)
    b = _run(tracer, scene, "warp", monkeypatch)
    assert np.array_equal(a.image, b.image) and np.array_equal(a.hit_sum, b.hit_sum)


@pytest.mark.parametrize("name,scale", [("bos", 0.02), ("tomo", 0.003)])
def test_default_variant_is_render_emitters(tracer, name, scale, monkeypatch):
    """render_emitters is the default for every scene; the call reports which
    kernel ran."""
    from paper_1812_05902_b200 import scenes
    monkeypatch.delenv("RAYBOS_K1", raising=False)
    scene, grid, info, desc = scenes.build(name, scale=scale)
    tracer.set_field(grid)
    assert tracer.run_trace(scene, True, True).report["k1_kernel"] == 1
