"""Prints the sweep lines of the last gpurun call (dev aid)."""
import json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "gpurun_out", ".last_call.json")))
print(d["status"], d["rc"], d.get("run_s"))
for l in d["stdout_tail"].splitlines():
    if "{" in l:
        pre, js = l.split("{", 1)
        j = json.loads("{" + js)
        print(pre, j["lib"], " ".join(f"{k}:{v['rays_per_s']:.4g}" for k, v in j.items() if k != "lib"))
    else:
        print(l[:300])
