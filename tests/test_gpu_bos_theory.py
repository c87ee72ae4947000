"""BOS displacement-vs-theory metrics at the BASELINE BOS shape (configs[1]:
20,480 dots x 1e4 rays through the 256^3 BDT-like field): the reference's own
metric chain (measure_dot_displacements -> grid_displacements ->
theoretical_displacement -> compare_fields, bos.cpp:97-244, via the test-only
ref shim) applied to the B200's rb_trace_bos_pair stats must reproduce the
metrics the unmodified reference produced from its own CPU traces (committed:
profiles/r02_bos_theory_reference_stats.npz, 70 min on 8 cores) within 1e-3
relative, with the same node count and the same valid dots
(scripts/bos_theory_check.py)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_STATS = os.path.join(ROOT, "profiles", "r02_bos_theory_reference_stats.npz")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libraybos_ref.so")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_bos_metrics_match_reference_at_baseline_shape(tmp_path):
    out = tmp_path / "bos_theory.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "bos_theory_check.py"),
                        "gpu", REF_STATS, str(out)], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep["same_scene_as_reference"] and rep["node_count_equal"]
    assert rep["valid_dots_identical"]
    assert max(rep["metrics_rel_diff"][k] for k in ("rms_error", "peak_abs_error", "pearson",
                                                    "peak_measured")) < 1e-3
    assert rep["max_dot_displacement_diff_px"] < 1e-3
