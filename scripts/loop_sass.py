"""Prints the spill instructions (with context) of K1's GRIN loop for one
render_emitters instantiation (dev aid).  usage: loop_sass.py lib.so ILb0ELi2E"""
import re, subprocess, sys
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
fn = sys.argv[2]
m = re.search(r"Function : \S*render_emitters" + fn, sass)
body = sass[m.start():]
body = body[:body.index("Function :", 20)] if "Function :" in body[20:] else body
lines = [l for l in body.splitlines() if re.match(r'\s+/\*[0-9a-f]{4,5}\*/', l)]
addr = [int(re.match(r'\s+/\*([0-9a-f]+)\*/', l).group(1), 16) for l in lines]
for i, l in enumerate(lines):
    m = re.search(r'BRA\s+(?:`\()?0x([0-9a-f]+)', l)
    if m and int(m.group(1), 16) < addr[i]:
        t = int(m.group(1), 16)
        region = [x for x, a in zip(lines, addr) if t <= a <= addr[i]]
        if any('LDG.E.128' in x for x in region) and 200 < len(region) < 1200:
            print(f"loop {hex(t)}-{hex(addr[i])}: {len(region)} instr")
            for j, x in enumerate(region):
                if 'STL' in x or 'LDL' in x:
                    for y in region[max(0, j - 4):j + 2]:
                        print("   ", y.strip()[:90])
                    print("   ---")
