"""The reference's own acceptance gate (tests/acceptance_main.cpp, 10 criteria:
Snell, RK4 order, null test, BOS uniform / blob, lens focus, sensor energy,
diffraction, bitwise PGM determinism, throughput floor) with its run_trace call
sites routed to the B200 drop-in: engine.cpp:511 (render) and 539-540 (bos_run)
go through raybos_gpu::run_trace / run_trace_bos_pair, acceptance_main.cpp:141,146
through raybos_gpu::run_trace.  oracle/route_drop_in.sh + oracle/Makefile build
it in the build container; the binary travels to the GPU box with the repo."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/acceptance_gpu not built")
def test_reference_acceptance_gate_through_drop_in():
    env = dict(os.environ, RAYBOS_GPUS="1")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "acceptance_gpu.log"), "w") as f:
        f.write(out)
    passed = re.findall(r"^\[PASS\] criterion\s+(\d+)", out, flags=re.M)
    assert r.returncode == 0, out
    assert sorted(int(p) for p in passed) == list(range(1, 11)), out
    assert "acceptance: all criteria passed" in out
