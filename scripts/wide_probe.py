import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from golden_io import load
from oracle.oracle import COracle
from paper_1812_05902_b200 import abi
from paper_1812_05902_b200.engine import GpuTracer
t = GpuTracer(1)
scene, field, g = load("blob")
scene.d_tau *= 3.0
t.set_field(field)
a = t.run_trace(scene, True, True)
b = COracle().trace(scene, field, True, True)
e = a.image - b.image
print("sum", a.image.sum(), b.image.sum(), "diff", e.sum())
print("edge rows/cols diff", e[:2].sum(), e[-2:].sum(), e[:, :2].sum(), e[:, -2:].sum(), "interior", e[2:-2, 2:-2].sum())
# per-source: trace each source alone
for d in range(6):
    sub = scene.subset([d])
    aa = t.run_trace(sub, True, True).image; bb = COracle().trace(sub, field, True, True).image
    print(d, sub.sources[0][:2], aa.sum(), bb.sum(), (aa.sum()-bb.sum())/max(bb.sum(),1e-30))
sub = scene.subset([4])
aa = t.run_trace(sub, True, True).image; bb = COracle().trace(sub, field, True, True).image
d = aa - bb
nz = np.argwhere(bb > 0)
r0, c0 = nz.min(0); r1, c1 = nz.max(0)
print("window rows", r0, r1, "cols", c0, c1)
print("row sums diff", np.round(d.sum(1)[r0:r1+1] / bb.sum() * 1e7, 2))
print("col sums diff", np.round(d.sum(0)[c0:c1+1] / bb.sum() * 1e7, 2))
print("gpu-only pixels", np.sum((aa > 0) & (bb == 0)), "ref-only", np.sum((bb > 0) & (aa == 0)))
