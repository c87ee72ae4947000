"""SURVEY §8(f) rows on the GPU: f4 trace_debug records (engine.cpp:605-624) and
f3 the render tail's quantize (sensor.cpp:124-135) computed on device."""
import numpy as np
import pytest

from golden_io import NAMES, load

pytestmark = pytest.mark.gpu

FIELD_FIXTURES = [n for n in NAMES if "debug_rays" in load(n)[2]]


@pytest.mark.parametrize("name", FIELD_FIXTURES)
def test_trace_debug_records_match_reference(tracer, name):
    scene, field, g = load(name)
    tracer.set_field(field)
    for k, (dot, ray) in enumerate(g["debug_rays"]):
        ref = g[f"debug_{k}"]
        got = tracer.trace_debug(scene, int(dot), int(ray))
        assert got.shape == ref.shape
        # FP64 validation arithmetic: bit-exact unless glibc's sin/cos of this ray's
        # aperture angle is not correctly rounded (test_sincos_rounding.py)
        scale = np.abs(ref).max(axis=0).clip(1e-30)
        assert (np.abs(got - ref) / scale).max() < 1e-13
        assert np.all(np.diff(got[:, 0]) > 0)  # xi increases (test_engine.cpp:217-221)


def test_trace_debug_errors(tracer):
    scene, field, g = load("small")
    tracer.set_field(field)
    with pytest.raises(Exception, match="dot index out of range"):
        tracer.trace_debug(scene, 9999, 0)
    with pytest.raises(Exception, match="ray index out of range"):
        tracer.trace_debug(scene, 0, 9999)
    tracer.set_field(None)
    with pytest.raises(Exception, match="no density field"):
        tracer.trace_debug(scene, 0, 0)


@pytest.mark.parametrize("name", ["small", "singlet_defocus", "blob"])
@pytest.mark.parametrize("bits", [16, 12, 8])
def test_device_quantize_matches_host_quantize(tracer, name, bits):
    from paper_1812_05902_b200 import setup as S
    scene, field, g = load(name)
    tracer.set_field(field)
    gain = 0.9 * ((1 << bits) - 1) / g["image_1"].max()
    res = tracer.run_trace(scene, True, True, quantize=(bits, gain))
    # same FP64 image -> identical counts (llround, clamp), as render would write them
    assert np.array_equal(res.quantized, S.quantize(res.image, bits, gain))
    # and within one count of quantizing the reference's own image
    ref_q = S.quantize(g["image_1"], bits, gain).astype(np.int64)
    assert np.abs(res.quantized.astype(np.int64) - ref_q).max() <= 1


@pytest.mark.parametrize("name", ["small", "blob", "field3d", "shock_particles"])
def test_bos_pair_equals_two_traces(tracer, name):
    """f2: rb_trace_bos_pair == rb_trace(no field) + rb_trace(field), bit for bit,
    and the per-dot displacement (measure_dot_displacements, bos.cpp:97-112)
    matches the reference's within 1e-3 px."""
    scene, field, g = load(name)
    tracer.set_field(field)
    ref_leg, grad_leg = tracer.trace_bos_pair(scene)
    a = tracer.run_trace(scene, False, False)
    b = tracer.run_trace(scene, True, False)
    for x, y in ((ref_leg, a), (grad_leg, b)):
        assert np.array_equal(x.hit_sum, y.hit_sum) and np.array_equal(x.landed, y.landed)
        for k in ("emitted", "landed", "lost", "blocked_aperture", "blocked_miss", "blocked_tir",
                  "blocked_sensor_miss"):
            assert x.report[k] == y.report[k], k
    m = (ref_leg.landed > 0) & (grad_leg.landed > 0)
    disp = grad_leg.hit_sum[m] / grad_leg.landed[m, None] - ref_leg.hit_sum[m] / ref_leg.landed[m, None]
    disp_ref = g["hit_sum_1"][m] / g["landed_1"][m, None] - g["hit_sum_0"][m] / g["landed_0"][m, None]
    assert np.abs(disp - disp_ref).max() / scene.sensor.pitch < 1e-3


@pytest.mark.parametrize("name", ["blob", "field3d", "shock_particles", "uniform_random"])
def test_cell_table_is_bit_identical(tracer, name, monkeypatch):
    """The per-cell coefficient table (capi.cpp build_cell_table) and the
    in-loop derivation from the nodes give the same bits: images, hits, steps,
    and the per-ray replay."""
    scene, field, g = load(name)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RAYBOS_CELL_TABLE", flag)
        tracer.set_field(field)
        nodes = tracer.field_bytes()
        res = tracer.run_trace(scene, True, True)
        src = np.repeat(np.arange(scene.n_sources), 3)
        ray = np.tile([0, scene.rays_per_source // 2, scene.rays_per_source - 1], scene.n_sources)
        out[flag] = (nodes, res, tracer.trace_rays(scene, src, ray))
    (b1, r1, t1), (b0, r0, t0) = out["1"], out["0"]
    assert b1 > b0  # the table was built (and only in the first pass)
    assert np.array_equal(r1.image, r0.image)
    assert np.array_equal(r1.hit_sum, r0.hit_sum) and np.array_equal(r1.landed, r0.landed)
    assert r1.report["total_steps"] == r0.report["total_steps"]
    for a, b in zip(t1, t0):
        assert np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


@pytest.mark.parametrize("name", ["blob", "shock_particles", "small"])
def test_emitter_split_is_invisible(tracer, name, monkeypatch):
    """Splitting an emitter over several CTAs (capi.cpp emitter_split) leaves the
    image, the landed counts and the DotHitStats sums (fixed point, kernels.cu
    kHitScale) bit-identical, bos pair mode included."""
    scene, field, g = load(name)
    tracer.set_field(field)
    runs = {}
    for split in ("1", "3", "8"):
        monkeypatch.setenv("RAYBOS_SPLIT", split)
        runs[split] = (tracer.run_trace(scene, True, True), tracer.trace_bos_pair(scene))
    (r1, p1) = runs["1"]
    for split in ("3", "8"):
        r, p = runs[split]
        assert np.array_equal(r.image, r1.image)
        assert np.array_equal(r.landed, r1.landed)
        drop = ("kernel_ms", "wall_seconds", "kernel_launches")
        assert {k: v for k, v in r.report.items() if k not in drop} == \
            {k: v for k, v in r1.report.items() if k not in drop}
        assert np.array_equal(r.hit_sum, r1.hit_sum)
        for a, b in zip(p, p1):
            assert np.array_equal(a.landed, b.landed)
            assert np.array_equal(a.hit_sum, b.hit_sum)


def test_kernel_launch_count_is_reported(tracer, monkeypatch):
    """rb_trace_out.kernel_launches: render (+ the chunk-stats kernel when
    emitters are split) (+ image finalize for rb_trace)."""
    scene, field, g = load("shock_particles")
    tracer.set_field(field)
    monkeypatch.setenv("RAYBOS_SPLIT", "1")
    assert tracer.run_trace(scene, True, True).report["kernel_launches"] == 2
    assert tracer.run_trace(scene, True, False).report["kernel_launches"] == 1
    monkeypatch.setenv("RAYBOS_SPLIT", "4")
    assert tracer.run_trace(scene, True, True).report["kernel_launches"] == 3


def test_large_grid_cell_table_matches_nodes(tracer, monkeypatch):
    """Config 5's 1024^3 grid (17 GB of nodes + a 137 GB cell table on one
    B200): 32-bit cell / node indexing and the table build at full size give
    the node path's bits on sampled rays, through real deflections."""
    from paper_1812_05902_b200 import scenes
    scene, grid, info, desc = scenes.build("large", scale=0.002)
    rng = np.random.default_rng(3)
    src = rng.integers(0, scene.n_sources, 2048)
    ray = rng.integers(0, scene.rays_per_source, 2048).astype(np.int32)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("RAYBOS_CELL_TABLE", flag)
        tracer.set_field(grid)
        out[flag] = (tracer.field_bytes(), tracer.trace_rays(scene, src, ray, True))
    (b1, (uv1, st1, n1)), (b0, (uv0, st0, n0)) = out["1"], out["0"]
    tracer.set_field(None)
    assert b1 > 100e9 and b0 == 1024 ** 3 * 16
    assert np.array_equal(st1, st0) and np.array_equal(n1, n0)
    assert np.array_equal(uv1, uv0, equal_nan=True)
    free, _ = tracer.trace_rays(scene, src, ray, False)[:2]
    ok = st1 == 0
    assert np.abs(uv1[ok] - free[ok]).max() / scene.sensor.pitch > 0.1  # the medium deflects
