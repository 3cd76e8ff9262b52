"""Registers / stack per kernel of the built library:  python tools/resources.py [regex]"""
import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parents[1] / "paper_1409_8116_b200" / "lib" / "libfastpoisson_b200.so"
txt = subprocess.run(["cuobjdump", "--dump-resource-usage", str(lib)], capture_output=True, text=True).stdout
names, rows = [], []
cur = None
for line in txt.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), int(m.group(2))))
        cur = None
dem = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
for (mang, reg, stack), d in sorted(zip(rows, dem), key=lambda x: x[1]):
    d = d.replace("void fpb::", "").replace("(fpb::FftPass)", "")
    if pat is None or pat.search(d):
        print(f"{d:60s} reg={reg:3d} stack={stack}")
