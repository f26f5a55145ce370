"""Summarise an ncu source page (cuda,sass CSV) by source line: stall samples,
executed instructions and the dominant stall reasons.

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
  python scripts/ncu_lines.py X.csv [top]
"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
agg = {}
hdr = None
fname = ""
for r in rows:
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
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
    except ValueError:
        continue
    stalls = {}
    for k, v in d.items():
        if k.startswith("stall_") or "Stall" in k and "Sampling" not in k:
            try:
                stalls[k] = int(v)
            except ValueError:
                pass
    try:
        ins = int(d.get("Instructions Executed", "0"))
    except ValueError:
        ins = 0
    key = (fname, int(r[0]), r[1].strip()[:80])
    a = agg.setdefault(key, [0, 0, {}])
    a[0] += s
    a[1] += ins
    for k, v in stalls.items():
        a[2][k] = a[2].get(k, 0) + v
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot}, instructions {toti}")
sort_i = 1 if len(sys.argv) > 3 and sys.argv[3] == "ins" else 0
for k, v in sorted(agg.items(), key=lambda x: -x[1][sort_i])[:top]:
    st = sorted(v[2].items(), key=lambda x: -x[1])[:3]
    sts = ", ".join(f"{n.replace('stall_', '')}={c}" for n, c in st if c)
    print(f"{v[0] / tot * 100:5.1f}% ins {v[1] / toti * 100:5.1f}%  {k[0]}:{k[1]:<4} {k[2]}  [{sts}]")
