"""Cull audit over whole workloads with the checked build.

The checked library (-DPSG_CHECKS) re-tests every candidate that the per-pixel
footprint rect or the fp32 homography cull rejects with the exact fp64 test
(eval_candidate's expression sequence) and counts acceptances as cull misses;
the z-bound counter checks the depth-bound early exit on every accepted
candidate. Both must be 0.

  PSG_LIB=paper_2412_03451_b200/lib/libpsplat_b200_checks.so \
    python scripts/cull_audit.py --config c3 --lams 7.3576,20,300 [--views N] [--stride S]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--lams", default="7.3576,20,300")
    ap.add_argument("--views", type=int, default=0, help="0 = all views of the workload")
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--precision", default="fp64")
    a = ap.parse_args()
    from paper_2412_03451_b200 import ViewBatch, _lib, scenes
    if not _lib.LIB_PATH.endswith("_checks.so"):
        sys.exit("cull_audit needs PSG_LIB=<...>/libpsplat_b200_checks.so")
    wl = scenes.load(a.config)
    picks = list(range(0, wl.n_views, a.stride))
    if a.views:
        picks = picks[:a.views]
    out = {"config": a.config, "views": len(picks), "stride": a.stride, "precision": a.precision,
           "library": os.path.basename(_lib.LIB_PATH), "lambdas": {}}
    vb = ViewBatch(precision=a.precision)
    vb.set_scene(wl.scene)
    vb.set_views([wl.cams[k] for k in picks])
    vb.render_ground_truth(wl.faces)
    for lam in (float(x) for x in a.lams.split(",")):
        vb.reset_stats()
        t0 = time.perf_counter()
        for b0 in range(0, len(picks), a.batch):
            ids = np.arange(b0, min(len(picks), b0 + a.batch))
            vb.zero_grads()
            vb.step(ids, lam, 1.0 / len(ids))
            vb.finalize()
            g, _ = vb.read_grads()
            assert np.isfinite(g).all()
        st = vb.stats()
        out["lambdas"][f"{lam:g}"] = {k: st[k] for k in ("pixel_pairs", "live_records", "cull_checks",
                                                         "cull_misses", "zbound_violations", "big_tiles")}
        out["lambdas"][f"{lam:g}"]["seconds"] = time.perf_counter() - t0
    out["ok"] = all(v["cull_misses"] == 0 and v["zbound_violations"] == 0 and v["cull_checks"] > 0
                    for v in out["lambdas"].values())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
