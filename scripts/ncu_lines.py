"""Per-CUDA-source-line instruction and stall profile of an ncu report (dev aid).
usage: python scripts/ncu_lines.py rep.ncu-rep [units] [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, hdr, agg = "?", None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit() or r[2] != "-":
        continue
    key = (fname, int(r[0]))
    ex = int(r[hdr["Instructions Executed"]] or 0)
    th = int(r[hdr["Thread Instructions Executed"]] or 0)
    sm = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    a = agg.setdefault(key, [0, 0, 0, r[1].strip()[:70]])
    a[0] += ex; a[1] += th; a[2] += sm
tex = sum(a[0] for a in agg.values()); tth = sum(a[1] for a in agg.values())
tsm = sum(a[2] for a in agg.values())
print(f"thread instr per unit {tth / units:.1f}; warp instr {tex:.3e}; samples {tsm}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:13s}{k[1]:5d} thr/unit {a[1] / units:8.1f} {a[1] / tth * 100:5.1f}%  stall {a[2] / max(tsm, 1) * 100:5.1f}%  {a[3]}")
