"""The N>1 path on CPU: world_size-2 gloo ranks each render their shard of the
emitters (rb_plan_shards) as a 64-bit fixed-point partial image — the same
integer accumulation the GPU kernel uses, computed here by the oracle — then
one all-reduce sums the partial images.  The result must be bit-identical to
the single-process render, as must the gathered per-emitter stats."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from golden_io import load
    from oracle.oracle import COracle
    from paper_1812_05902_b200.engine import plan_shards
    scene, field, g = load(name)
    plan = plan_shards(scene, world)
    res = COracle().trace(scene, field, True, True, shard_of=plan, shard_index=rank,
                          fixed_point=True)
    img = torch.from_numpy(res.fixed.astype(np.int64).ravel())
    dist.all_reduce(img)                                   # the one exchange step
    hit = torch.from_numpy(res.hit_sum.copy())
    landed = torch.from_numpy(res.landed.copy())
    dist.all_reduce(hit)                                   # disjoint owners: exact
    dist.all_reduce(landed)
    counters = torch.tensor([res.report[k] for k in ("emitted", "landed", "lost",
                                                     "blocked_aperture")], dtype=torch.int64)
    dist.all_reduce(counters)
    if rank == 0:
        np.savez(os.path.join(out_dir, "out.npz"), img=img.numpy(), hit=hit.numpy(),
                 landed=landed.numpy(), counters=counters.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["blob", "singlet_defocus"])
def test_two_rank_shard_and_reduce_is_bit_identical(tmp_path, oracle, name):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_io import load
    port = _free_port()
    mp.spawn(_worker, args=(2, port, name, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "out.npz")
    scene, field, g = load(name)
    full = oracle.trace(scene, field, True, True, fixed_point=True)
    assert np.array_equal(got["img"], full.fixed.astype(np.int64).ravel())
    assert np.array_equal(got["hit"], full.hit_sum)
    assert np.array_equal(got["landed"], full.landed)
    r = full.report
    assert list(got["counters"]) == [r["emitted"], r["landed"], r["lost"], r["blocked_aperture"]]
    # and the fixed-point image is the FP64 reference image to within the quantum
    ref = g["image_1"].ravel()
    fx = got["img"] / 2.0 ** 31
    assert np.linalg.norm(fx - ref) / np.linalg.norm(ref) < 1e-6
