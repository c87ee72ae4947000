"""Loads the reference-generated fixtures of tests/golden (see make_golden.py)."""
import json
import os

import numpy as np

from paper_1812_05902_b200.scene import FieldNodes, FlatScene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


def load(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    scene = FlatScene.from_json(json.loads(str(d["scene_json"])))
    field = None
    if "field_n" in d:
        nx, ny, nz = (int(v) for v in d["field_dims"])
        field = FieldNodes(nx, ny, nz, tuple(d["field_origin"]), tuple(d["field_spacing"]),
                           d["field_n"], d["field_gx"], d["field_gy"], d["field_gz"])
    return scene, field, d
