"""Turn the round's ncu outputs into the committed summaries under profiles/.

  python scripts/summarize_ncu.py --tag r1 --launches gpurun_out/launches_r1.csv \
      --full gpurun_out/bench_raster_full.ncu-rep --config c3 --views 1024 --lam 300 \
      --precision fp64

Writes profiles/<tag>_launches.csv (raw launch list), profiles/<tag>_launch_shares.txt,
profiles/<tag>_raster_full.txt (key counters + per-line stall hot spots) and
profiles/raster_dram_bytes.json (DRAM bytes per rasteriser launch, read by bench.py
as roofline.traffic when its config matches).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__grid_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
]


def launch_shares(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0].strip()[:90]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    s = sum(tot.values())
    out = ["share     total_us       launches  kernel (ncu gpu__time_duration, cold/serialised)"]
    for k, v in tot.most_common():
        out.append(f"{v / s * 100:6.2f}%  {v:12.1f}  {cnt[k]:8d}   {k}")
    return "\n".join(out) + "\n"


def ncu_csv(rep: str, *args) -> str:
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--views", type=int, default=1024)
    ap.add_argument("--lam", type=float, default=300.0)
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--what", default="first rasteriser launch of bench.py")
    ap.add_argument("--phasemap", help="phase map JSON of the captured source (default: derived from "
                                       "the current psg_raster.cu by scripts/phasemap.py)")
    ap.add_argument("--no-traffic-json", action="store_true",
                    help="do not update raster_dram_bytes.json (captures other than the bench's)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        shutil.copy(a.launches, os.path.join(PROF, f"{a.tag}_launches.csv"))
        with open(os.path.join(PROF, f"{a.tag}_launch_shares.txt"), "w") as f:
            f.write(launch_shares(a.launches))
    if a.full:
        raw = list(csv.reader(io.StringIO(ncu_csv(a.full, "--page", "raw"))))
        hdr, units, vals = raw[0], raw[1], raw[2]
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines = [f"ncu --set full capture: {os.path.basename(a.full)} ({a.what}, "
                 f"{a.config}, {a.views} views, lambda={a.lam}, {a.precision})", ""]
        for k in KEYS:
            lines.append(f"{k:70s} {d.get(k, 'n/a'):>20s} {u.get(k, '')}")

        def to_bytes(k):
            v = float(d[k].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u[k]]
            return v * mult

        traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
        lines += ["", f"DRAM traffic per launch: {traffic / 1e9:.3f} GB "
                      f"({traffic / a.views / 1e6:.3f} MB per view)", ""]
        src = ncu_csv(a.full, "--page", "source", "--print-source", "cuda,sass")
        tmp = os.path.join(PROF, ".tmp_src.csv")
        with open(tmp, "w") as f:
            f.write(src)
        hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), tmp, "30"],
                             capture_output=True, text=True).stdout
        # executed warp instructions, lanes and stall samples per phase of the
        # rasteriser (source-derived line ranges, scripts/phasemap.py)
        pm = os.path.join(PROF, ".tmp_phasemap.json")
        with open(pm, "w") as f:
            if a.phasemap:
                f.write(open(a.phasemap).read())
            else:
                f.write(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "phasemap.py")],
                                       capture_output=True, text=True).stdout)
        phases = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_phases.py"), tmp, pm,
                                 "--views", str(a.views)], capture_output=True, text=True).stdout
        os.remove(tmp)
        os.remove(pm)
        lines += ["Per-phase breakdown (SASS instructions attributed to source lines; shared helper",
                  "lines inherit the phase of the surrounding code; M inst/view on the source-page",
                  "count basis, which runs ~10 % above smsp__inst_executed):", phases,
                  "Stall-sample hot spots by source line:", hot]
        with open(os.path.join(PROF, f"{a.tag}_raster_full.txt"), "w") as f:
            f.write("\n".join(lines))
        if a.no_traffic_json:
            return
        with open(os.path.join(PROF, "raster_dram_bytes.json"), "w") as f:
            def num(k):
                try:
                    return float(d[k].replace(",", ""))
                except (KeyError, ValueError):
                    return None

            counters = {
                "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "pipe_fp64_pct": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                "pipe_lsu_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                "pipe_alu_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                "pipe_fma_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                "threads_per_warp_inst": num("smsp__thread_inst_executed_per_inst_executed.ratio"),
                "local_ld_l1_hit_pct": num("l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct"),
                "shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                "red_sectors_l2": num("lts__t_sectors_srcunit_tex_op_red.sum"),
            }
            json.dump({"config": a.config, "views": a.views, "lambda": a.lam,
                       "precision": a.precision, "dram_bytes_per_launch": traffic,
                       "counters": counters,
                       "source": f"profiles/{a.tag}_raster_full.txt"}, f, indent=1)


if __name__ == "__main__":
    main()
