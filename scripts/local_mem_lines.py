"""Attribute local-memory traffic (ncu "L2 Theoretical Sectors Local") to source
lines of a `--set full --import-source on` capture.

  python scripts/local_mem_lines.py X.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname, agg = None, "", {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def f(k):
        try:
            return float(d.get(k, "0") or 0)
        except ValueError:
            return 0.0
    loc = f("L2 Theoretical Sectors Local")
    if loc > 0:
        a = agg.setdefault((fname, int(r[0]), r[1].strip()[:90]), [0.0, 0.0, 0.0])
        a[0] += loc
        a[1] += f("Instructions Executed")
        a[2] += f("Thread Instructions Executed")
tot = sum(a[0] for a in agg.values()) or 1.0
print(f"local-memory L2 theoretical sectors: {tot:.4g}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{a[0] / tot * 100:5.1f}%  sectors/inst {a[0] / max(a[1], 1):5.1f}  threads/inst "
          f"{a[2] / max(a[1], 1):5.1f}  {k[0]}:{k[1]}  {k[2]}")
