"""One rank of a one-process-per-GPU job (tests/test_gpu_multi.py):

    rank_worker.py <uid hex> <rank> <world> <fixture> <out.npz> trace|pair

Creates its context with rb_create_rank on $RAYBOS_RANK_DEVICE, renders the
fixture through rb_trace (or rb_trace_bos_pair) and saves what it returned."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def main():
    uid, rank, world, name, out, mode = sys.argv[1:7]
    rank, world = int(rank), int(world)
    from golden_io import load
    from paper_1812_05902_b200.engine import GpuTracer
    scene, field, _ = load(name)
    t = GpuTracer.for_rank(int(os.environ.get("RAYBOS_RANK_DEVICE", "0")), rank, world,
                           bytes.fromhex(uid))
    info = t.comm_info()
    t.set_field(field)
    if mode == "pair":
        r0, r1 = t.trace_bos_pair(scene)
        np.savez(out, hit_sum=r1.hit_sum, landed=r1.landed, hit_sum0=r0.hit_sum,
                 landed0=r0.landed, **info)
    else:
        res = t.run_trace(scene, with_field=True, accumulate_image=True,
                          host_image=(rank == 0))
        rep = res.report
        np.savez(out, hit_sum=res.hit_sum, landed=res.landed,
                 image=res.image if res.image is not None else np.zeros(0),
                 emitted=rep["emitted"], lost=rep["lost"], total_steps=rep["total_steps"],
                 threads=rep["threads"], **info)
    t.close()


if __name__ == "__main__":
    main()
