"""GPU vs oracle image error structure on a reference builtin scene (dev aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from oracle.oracle import COracle
from paper_1812_05902_b200.engine import GpuTracer
import json
d = np.load(sys.argv[1], allow_pickle=True)
from paper_1812_05902_b200.scene import FlatScene, FieldNodes
sc = FlatScene.from_json(json.loads(str(d["scene_json"])))
f = FieldNodes(*[int(x) for x in d["dims"]], tuple(d["origin"]), tuple(d["spacing"]), d["n"], d["gx"], d["gy"], d["gz"])
t = GpuTracer(1); t.set_field(f)
g = t.run_trace(sc, True, True)
o = COracle().trace(sc, f, True, True)
e = g.image - o.image
print("rel L2", np.linalg.norm(e) / np.linalg.norm(o.image), "max abs", np.abs(e).max(), "max val", o.image.max())
print("sum gpu", g.image.sum(), "sum ref", o.image.sum(), "landed eq", np.array_equal(g.landed, o.landed))
idx = np.unravel_index(np.argsort(-np.abs(e).ravel())[:10], e.shape)
for r, c in zip(*idx): print(r, c, o.image[r, c], g.image[r, c], e[r, c])
# error by column/row margin
print("err near edges", np.linalg.norm(e[:, :6]), np.linalg.norm(e[:, -6:]), np.linalg.norm(e[6:-6, 6:-6]))
