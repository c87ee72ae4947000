"""Host-side API details of rb_trace: the cached shard plan (reused only for
bit-identical sources; rb_plan_reset forces a re-plan) and page-locked output
buffers (rb_host_alloc)."""
import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


def test_plan_cache_is_invisible_and_resettable(tracer):
    scene, field, g = load("blob")
    tracer.set_field(field)
    a = tracer.run_trace(scene)
    b = tracer.run_trace(scene)                    # cached plan, device sources reused
    tracer.reset_plan()
    c = tracer.run_trace(scene)                    # re-planned and re-uploaded
    for r in (b, c):
        assert np.array_equal(r.image, a.image) and np.array_equal(r.hit_sum, a.hit_sum)
    # same count, one source moved: the cache must notice (memcmp of the sources)
    moved = scene.subset(np.arange(scene.n_sources))
    moved.source_ids = None
    moved.sources = scene.sources.copy()
    moved.sources[3, 0] += 1e-4
    d = tracer.run_trace(moved)
    ref = tracer.run_trace(moved)
    assert not np.array_equal(d.hit_sum[3], a.hit_sum[3])
    assert np.array_equal(d.hit_sum, ref.hit_sum)
    e = tracer.run_trace(scene)
    assert np.array_equal(e.image, a.image)


def test_pinned_image_out(tracer):
    scene, field, g = load("small")
    tracer.set_field(field)
    ref = tracer.run_trace(scene)
    buf = tracer.pinned((scene.height, scene.width))
    got = tracer.run_trace(scene, image_out=buf)
    assert got.image is buf and np.array_equal(buf, ref.image)
