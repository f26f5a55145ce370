"""Per-phase breakdown of executed warp instructions, thread instructions and stall
samples of one kernel, from an ncu source page exported with SASS:

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
  python scripts/ncu_phases.py X.csv PHASEMAP.json [--views N]

Each SASS instruction belongs to the source line it is listed under. Lines that
name a phase (ranges in PHASEMAP, psg_raster.cu line numbers of the captured
build) set the phase; instructions of shared helpers (dmul/dadd, intrinsics
headers) inherit the phase of the nearest preceding phase-specific instruction
in address order, which follows the compiler's block layout of the inlined code.
"""
import argparse
import csv
import json
import os

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("phasemap")
ap.add_argument("--views", type=float, default=0)
ap.add_argument("--file", default="psg_raster.cu")
a = ap.parse_args()

pm = json.load(open(a.phasemap))
ranges = [(int(lo), int(hi), name) for name, rs in pm.items() for lo, hi in rs]


def phase_of(fname, line):
    """(range width, phase) of the narrowest range holding the line, or None."""
    if not fname.endswith(a.file):
        return None
    best = None
    for lo, hi, name in ranges:
        if lo <= line <= hi and (best is None or hi - lo < best[0]):
            best = (hi - lo, name)
    return best


rows = list(csv.reader(open(a.csv)))
fname, hdr, cur_line = "", None, None
inst = {}  # addr -> [best phase match, ins, thread_ins, stall]; an address listed under
# several lines (its inline stack) takes the narrowest phase range among them
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        cur_line = int(r[0])
        continue
    if r[0] == "" and r[2].startswith("0x"):
        try:
            ins = int(r[7])
            thr = int(r[8])
            st = int(r[4])
        except ValueError:
            continue
        ph = phase_of(fname, cur_line)
        e = inst.setdefault(int(r[2], 16), [None, ins, thr, st])
        if ph is not None and (e[0] is None or ph[0] < e[0][0]):
            e[0] = ph
agg = {}
cur = "other"
for addr in sorted(inst):
    ph, ins, thr, st = inst[addr]
    if ph is not None:
        cur = ph = ph[1]
    else:
        ph = cur
    e = agg.setdefault(ph, [0, 0, 0])
    e[0] += ins
    e[1] += thr
    e[2] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"{'phase':14s} {'warp-inst':>14s} {'share':>7s} {'lanes':>6s} {'stalls':>7s}" +
      (f" {'M inst/view':>12s}" if a.views else ""))
for ph, (ins, thr, st) in sorted(agg.items(), key=lambda x: -x[1][0]):
    lanes = thr / ins if ins else 0
    extra = f" {ins / a.views / 1e6:12.2f}" if a.views else ""
    print(f"{ph:14s} {ins:14d} {ins / ti * 100:6.1f}% {lanes:6.1f} {st / ts * 100:6.1f}%{extra}")
print(f"{'total':14s} {ti:14d}" + (f" {'':14s} {ti / a.views / 1e6:12.2f}" if a.views else ""))
