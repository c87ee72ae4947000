"""CPU checks of the round-2 host pieces: the NCCL stand-in used by the one-GPU
multi-device tests, the acceptance-gate routing recipe, and bench.py's launch
contract."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NCCL_SYMBOLS = ["ncclGetUniqueId", "ncclCommInitAll", "ncclCommInitRank", "ncclReduce",
                "ncclAllReduce", "ncclGroupStart", "ncclGroupEnd", "ncclCommDestroy",
                "ncclCommCount", "ncclGetVersion"]


def test_fake_nccl_exports_what_the_library_dlopens():
    from paper_1812_05902_b200 import build
    lib = build.build_fake_nccl()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (nccl\w+)", out))
    assert set(NCCL_SYMBOLS) <= exported
    # ... and these are exactly the entry points capi.cpp resolves
    src = open(os.path.join(ROOT, "paper_1812_05902_b200", "csrc", "capi.cpp")).read()
    resolved = set(re.findall(r'RB_SYM\(\w+, "(nccl\w+)"\)', src))
    assert resolved == set(NCCL_SYMBOLS)


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/src/engine.cpp"),
                    reason="reference sources absent")
def test_drop_in_routing_changes_exactly_the_documented_call_sites(tmp_path):
    subprocess.run(["sh", os.path.join(ROOT, "oracle", "route_drop_in.sh"),
                    "/root/reference/proj", str(tmp_path)], check=True)
    ref = open("/root/reference/proj/src/engine.cpp").read().splitlines()
    gen = open(tmp_path / "engine_gpu.cpp").read().splitlines()
    # the copy differs from the reference only at the include and the call sites
    # (render's one line; bos_run's two lines become the pair call + two moves)
    changed = [l for l in gen if l not in ref]
    removed = [l for l in ref if l not in gen]
    assert len(changed) == 5 and len(removed) == 3, (changed, removed)
    assert all(re.search(r"\brun_trace\(setup", l) for l in removed)
    assert sum(l.count("raybos_gpu::run_trace") for l in changed) == 4
    acc = open(tmp_path / "acceptance_gpu.cpp").read()
    assert acc.count("raybos_gpu::run_trace(") == 2


def test_bench_rejects_a_world_size_that_is_not_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_bench_traffic_scales_with_the_launch_and_spot_windows():
    import bench
    from paper_1812_05902_b200 import scenes
    t1 = bench.profiled_traffic("large", 2e7)
    t2 = bench.profiled_traffic("large", 5e8)
    if t1 is not None:
        assert abs(t2 / t1 - 25.0) < 1e-9
    scene, _, _, _ = scenes.build("piv")
    # PIV: d_tau 47.2 um, sigma = d_tau / 4, 4 sigmas each side at 10 um pitch
    hw = 4 * 0.25 * scene.d_tau / 1e-5
    assert abs(bench.spot_reds_per_ray(scene) - (2 * hw + 1) ** 2) < 1e-9
