"""Per-pixel work counters of the rasteriser (a -DPSG_PROBE build):
  PSG_LIB=_variants/libpsplat_b200_probe.so python scripts/probe_work.py [--config c3] [--views 32]"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["considered", "exact_tests", "exact_reject_full_list", "insertions", "mid_list_insertions",
         "shifts", "pixels_done_early", "pixels_full_list", "pixels", "exact_reject_free_list",
         "appends_dropped_full", "tile_candidates"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--views", type=int, default=32)
    ap.add_argument("--lams", default="7.3576,20,54,300")
    a = ap.parse_args()
    from paper_2412_03451_b200 import ViewBatch, scenes
    wl = scenes.load(a.config)
    picks = [int(k * wl.n_views // a.views) for k in range(a.views)]
    vb = ViewBatch(precision="fp64")
    vb.set_scene(wl.scene)
    vb.set_views([wl.cams[k] for k in picks])
    vb.render_ground_truth(wl.faces)
    out = {}
    for lam in (float(x) for x in a.lams.split(",")):
        for rep in range(2):  # the first step of a fresh context replays (capacity probe)
            vb.reset_stats()
            vb.zero_grads()
            vb.step(np.arange(len(picks)), lam, 1.0)
            vb.finalize()
        buf = (C.c_uint64 * 12)()
        vb.L.psg_debug_probe(vb.h, buf)
        v = dict(zip(NAMES, list(buf)))
        px = max(v["pixels"], 1)
        out[f"{lam:g}"] = {k: v[k] / px for k in NAMES if k != "pixels"}
        out[f"{lam:g}"]["pixels"] = px
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
