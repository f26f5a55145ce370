"""One fused step over a slice of a workload, for ncu captures and quick timing.

  python scripts/profile_step.py --config c3 --views 64 --lam 300 --precision fp32 --reps 3
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--views", type=int, default=64)
    ap.add_argument("--lam", default="300", help="comma-separated lambdas, run in order")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--maps", type=int, default=1)
    ap.add_argument("--backward", type=int, default=1)
    args = ap.parse_args()
    import torch

    from paper_2412_03451_b200 import ViewBatch, scenes

    wl = scenes.load(args.config)
    V = min(args.views, wl.n_views)
    vb = ViewBatch(precision=args.precision)
    s = torch.cuda.Stream()
    vb.set_stream(s.cuda_stream)
    vb.set_scene(wl.scene)
    vb.set_views(list(wl.cams)[:V])
    vb.render_ground_truth(wl.faces)
    ids = np.arange(V, dtype=np.int32)
    vb.set_timing(True)
    for r in range(args.reps * len(args.lam.split(","))):
        lam = float(args.lam.split(",")[r // args.reps])
        t0 = time.perf_counter()
        vb.zero_grads()
        vb.step(ids, lam, 1.0 / V, write_maps=bool(args.maps), backward=bool(args.backward))
        vb.finalize()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ms = vb.kernel_ms()
        print(f"lambda {lam:g} rep {r}: step {dt * 1e3:.2f} ms wall, raster {ms:.3f} ms "
              f"({V / (ms / 1e3):.0f} views/s raster-only), stats {vb.stats()}")


if __name__ == "__main__":
    main()
