"""The library's own multi-GPU paths (reference partition
invariance: engine.cpp:468-490, test_engine.cpp:105-127, acceptance_main.cpp:107-129).

rb_trace over several devices — in-process (rb_create / rb_create_devices, one
NCCL communicator per device) and one process per GPU (rb_create_rank) — must
return the image, per-source DotHitStats and RunReport counters of the
single-device call bit for bit, including when some devices own no sources.

On a box with one GPU these run the library's real multi-device code (shard
plan, per-device threads, the grouped collectives, the stats merge and
all-reduce) against tests/fake_nccl, a host-staged NCCL stand-in selected with
RAYBOS_NCCL_LIB: real NCCL refuses two ranks on one device, and collective
kernels of several ranks on one GPU must not wait on each other.  With two or
more GPUs the same checks also run against the real NCCL.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
FAKE = os.path.join(ROOT, "tests", "fake_nccl", "libfakenccl.so")

pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.fixture
def fake_nccl(monkeypatch, tmp_path):
    if not os.path.exists(FAKE):
        from paper_1812_05902_b200 import build
        build.build_fake_nccl()
    monkeypatch.setenv("RAYBOS_NCCL_LIB", FAKE)
    monkeypatch.setenv("RAYBOS_FAKE_NCCL_DIR", str(tmp_path))
    return FAKE


def _single(name, with_field=True):
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    scene, field, _ = load(name)
    with GpuTracer(n_devices=1) as t:
        t.set_field(field)
        return t.run_trace(scene, with_field=with_field, accumulate_image=True)


def _same(a, b):
    assert np.array_equal(a.landed, b.landed)
    assert np.array_equal(a.hit_sum, b.hit_sum)          # fixed-point sums: exact
    if a.image is not None or b.image is not None:
        assert np.array_equal(a.image, b.image)          # integer image: exact
    for k in ("emitted", "landed", "lost", "blocked_aperture", "blocked_miss", "blocked_tir",
              "blocked_sensor_miss", "total_steps"):
        assert a.report[k] == b.report[k], k


# small has 12 sources: with 2-3 devices all but device 0 own nothing (shards are
# dealt in tiles of 32) and must still join the reduce
CASES = ["small", "blob", "singlet_defocus", "shock_particles"]


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
@pytest.mark.parametrize("name", CASES)
def test_in_process_devices_bit_identical(fake_nccl, name, devices):
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    ref = _single(name)
    scene, field, _ = load(name)
    with GpuTracer(devices=devices) as t:
        assert t.n_devices == len(devices)
        info = t.comm_info()
        assert info["comm_ranks"] == len(devices) and info["world"] == 1
        t.set_field(field)
        got = t.run_trace(scene, with_field=True, accumulate_image=True)
        assert got.report["threads"] == len(devices)
        _same(got, ref)
        # stats-only call (no image, no image reduce) and the bos pair
        s = t.run_trace(scene, with_field=True, accumulate_image=False)
        assert np.array_equal(s.hit_sum, ref.hit_sum)
        if field is not None:
            r0, r1 = t.trace_bos_pair(scene)
            assert np.array_equal(r1.hit_sum, ref.hit_sum)
            assert np.array_equal(r1.landed, ref.landed)


def test_in_process_quantized_and_device_image(fake_nccl):
    import torch
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    scene, field, _ = load("blob")
    with GpuTracer(n_devices=1) as t1:
        t1.set_field(field)
        ref = t1.run_trace(scene, quantize=(12, 3.0))
    with GpuTracer(devices=[0, 0]) as t:
        t.set_field(field)
        fx = torch.zeros(scene.width * scene.height, dtype=torch.int64, device="cuda")
        got = t.run_trace(scene, quantize=(12, 3.0), image_fixed_ptr=fx.data_ptr())
        assert np.array_equal(got.quantized, ref.quantized)
        assert np.array_equal(fx.cpu().numpy() / 2.0 ** 31, ref.image.ravel())
        # quantized without an FP64 host image is still written
        q = t.run_trace(scene, quantize=(12, 3.0), host_image=False)
        assert q.image is None and np.array_equal(q.quantized, ref.quantized)


def _run_ranks(name, world, tmp_path, extra_env, pair=False):
    from paper_1812_05902_b200.engine import nccl_unique_id
    uid = nccl_unique_id()
    env = dict(os.environ, **extra_env)
    procs = []
    for r in range(world):
        out = tmp_path / f"rank{r}.npz"
        cmd = [sys.executable, os.path.join(ROOT, "tests", "rank_worker.py"), uid.hex(), str(r),
               str(world), name, str(out), "pair" if pair else "trace"]
        dev = r % _gpus()
        procs.append(subprocess.Popen(cmd, env=dict(env, RAYBOS_RANK_DEVICE=str(dev)),
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["blob", "small", "singlet_defocus"])
def test_rank_mode_bit_identical(fake_nccl, tmp_path, name, world):
    ref = _single(name)
    res = _run_ranks(name, world, tmp_path, {})
    for r, d in enumerate(res):
        assert int(d["comm_ranks"]) == world and int(d["world"]) == world
        # every rank returns the whole call's stats and counters (all-reduced)
        assert np.array_equal(d["landed"], ref.landed)
        assert np.array_equal(d["hit_sum"], ref.hit_sum)
        assert int(d["emitted"]) == ref.report["emitted"]
        assert int(d["lost"]) == ref.report["lost"]
        assert int(d["total_steps"]) == ref.report["total_steps"]
        assert int(d["threads"]) == world
    assert np.array_equal(res[0]["image"], ref.image)     # the image lands on rank 0
    assert res[1]["image"].size == 0


def test_rank_mode_bos_pair(fake_nccl, tmp_path):
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    scene, field, _ = load("blob")
    with GpuTracer(n_devices=1) as t:
        t.set_field(field)
        r0, r1 = t.trace_bos_pair(scene)
    res = _run_ranks("blob", 2, tmp_path, {}, pair=True)
    for d in res:
        assert np.array_equal(d["hit_sum"], r1.hit_sum) and np.array_equal(d["landed"], r1.landed)
        assert np.array_equal(d["hit_sum0"], r0.hit_sum) and np.array_equal(d["landed0"], r0.landed)


@pytest.mark.skipif("_gpus() < 2")
@pytest.mark.parametrize("name", CASES)
def test_real_nccl_all_devices_bit_identical(name):
    """rb_create(all visible GPUs) with the real NCCL: the drop-in's default on
    an 8-GPU node (RAYBOS_GPUS unset)."""
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    ref = _single(name)
    scene, field, _ = load(name)
    with GpuTracer(n_devices=0) as t:
        t.set_field(field)
        _same(t.run_trace(scene), ref)


@pytest.mark.skipif("_gpus() < 2")
def test_real_nccl_rank_mode(tmp_path):
    ref = _single("blob")
    res = _run_ranks("blob", 2, tmp_path, {"RAYBOS_NCCL_LIB": ""})
    assert np.array_equal(res[0]["image"], ref.image)
    assert np.array_equal(res[1]["hit_sum"], ref.hit_sum)


@pytest.mark.parametrize("name", ["blob", "small", "singlet_defocus", "shock_particles"])
def test_real_nccl_one_rank_job(monkeypatch, name):
    """rb_create_rank(world = 1) with an id builds a real one-rank NCCL
    communicator, so the rank-mode exchange (image ncclReduce + the all-reduces of
    stats, counters and error flag, grouped on the device stream) runs against the
    real libnccl on one GPU — nothing waits on another rank."""
    monkeypatch.delenv("RAYBOS_NCCL_LIB", raising=False)
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer, nccl_unique_id
    ref = _single(name)
    scene, field, _ = load(name)
    t = GpuTracer.for_rank(0, 0, 1, nccl_unique_id())
    try:
        info = t.comm_info()
        assert info["comm_ranks"] == 1 and info["world"] == 1 and info["nccl_version"] > 0
        t.set_field(field)
        _same(t.run_trace(scene), ref)
        if field is not None:
            with GpuTracer(1) as t1:
                t1.set_field(field)
                a0, a1 = t1.trace_bos_pair(scene)
            b0, b1 = t.trace_bos_pair(scene)
            assert np.array_equal(a0.hit_sum, b0.hit_sum) and np.array_equal(a1.hit_sum, b1.hit_sum)
    finally:
        t.close()


@pytest.mark.parametrize("name,scale", [("tomo", 0.005), ("bos", 0.02)])
def test_bench_scene_on_three_devices_bit_identical(fake_nccl, name, scale):
    """A bench scene (bos: emitter splitting, 4 CTAs per emitter),
    the cell table and the shard-plan cache, on three in-process devices."""
    from paper_1812_05902_b200 import scenes
    from paper_1812_05902_b200.engine import GpuTracer
    scene, grid, info, desc = scenes.build(name, scale=scale)
    with GpuTracer(n_devices=1) as t1:
        t1.set_field(grid)
        ref = t1.run_trace(scene)
    with GpuTracer(devices=[0, 0, 0]) as t:
        t.set_field(grid)
        for _ in range(2):                       # second call: cached plan on every device
            _same(t.run_trace(scene), ref)
