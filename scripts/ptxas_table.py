"""Registers / spills per raster kernel from the ptxas -v log of the build.

  python scripts/ptxas_table.py [paper_2412_03451_b200/csrc/_obj/raster_ptxas.log]
"""
import re
import subprocess
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "paper_2412_03451_b200/csrc/_obj/raster_ptxas.log"
lines = open(path).read().splitlines()
name = None
out = []
for i, l in enumerate(lines):
    m = re.search(r"Compiling entry function '([^']+)'", l)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"psg::\(anonymous namespace\)::", "", name)
        name = re.sub(r"\(.*", "", name)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", l)
    if m and name:
        regs = re.search(r"Used (\d+) registers", lines[i + 1])
        out.append((name, regs.group(1) if regs else "?", m.group(2), m.group(3)))
        name = None
for n, r, ss, sl in sorted(out):
    print(f"{n:45s} regs {r:>4s}  spill st {ss:>4s} ld {sl:>4s}")
