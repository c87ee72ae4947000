"""Per-instruction execution profile of an ncu report's SASS (dev aid).
usage: python scripts/sass_hot.py rep.ncu-rep [rays_steps]
Prints the instruction-class mix weighted by 'Instructions Executed' and the
hottest basic blocks."""
import csv, io, re, subprocess, sys, collections
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    ex = int(r[ix["Instructions Executed"]] or 0)
    th = int(r[ix["Thread Instructions Executed"]] or 0)
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    recs.append((r[ix["Address"]], src, ex, th, smp))
tot = sum(e for _, _, e, _, _ in recs)
tth = sum(t for _, _, _, t, _ in recs)
print(f"warp instr {tot:.4e}  thread instr {tth:.4e}")
if len(sys.argv) > 2:
    n = float(sys.argv[2])
    print(f"thread instr per unit {tth / n:.1f}   warp instr per unit*32 {tot * 32 / n:.1f}")
mix = collections.Counter()
for _, s, e, t, _ in recs:
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split(" ")[0]
    mix[op.split(".")[0]] += e
for op, e in mix.most_common(30):
    print(f"{op:10s} {e / tot * 100:6.2f}%")
# hottest instructions
print("--- hottest 60 instructions")
idx = sorted(range(len(recs)), key=lambda i: -recs[i][2])[:60]
for i in sorted(idx):
    a, s, e, t, smp = recs[i]
    print(f"{i:5d} {e:12d} {t / max(e, 1):5.1f} {smp:7d}  {s[:90]}")
