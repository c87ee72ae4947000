"""K1 under the bounds-checked build.  compute-sanitizer is closed
on this pool (profiles/r02_compute_sanitizer_closed.log), so the library is
built a second time with RB_CHECKED=1: every shared-memory tile / weight slot,
global image, cell-table, node-grid, work-order and stats-partial index K1
computes is range-checked on device, and a violation fails the call.  The
reference is race-free by construction (private per-worker buffers,
engine.cpp:442-447); K1's shared-tile atomics and work queue are covered by the
bit-reproducibility tests (any race would change an integer sum between runs,
splits or device counts: test_gpu_tail.py, test_gpu_multi.py)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1812_05902_b200", "libraybos_gpu_checked.so")

pytestmark = pytest.mark.gpu


def test_k1_has_no_out_of_range_access():
    if not os.path.exists(CHECKED):
        from paper_1812_05902_b200 import build
        build.build_checked_library()
    env = dict(os.environ, RAYBOS_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checked_worker.py")],
                       capture_output=True, text=True, timeout=1500, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    recs = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "checked_build.jsonl"), "w") as f:
        f.write(r.stdout)
    assert len(recs) >= 30
    for rec in recs:  # the checked kernels still compute: every split gives the same image
        assert rec["image_sum_split1"] == rec["image_sum_split3"], rec
        assert rec["landed_split1"] == rec["landed_split3"], rec
