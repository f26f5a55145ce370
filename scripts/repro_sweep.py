"""Debug helper: bench.py's step sequence (lambda 300 then 20) with options."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=1024)
    ap.add_argument("--timing", type=int, default=0)
    ap.add_argument("--n300", type=int, default=10)
    ap.add_argument("--lam2", type=float, default=20.0)
    ap.add_argument("--bench_seq", type=int, default=0, help="1: timing window + reset_stats + stats")
    a = ap.parse_args()
    import torch
    from paper_2412_03451_b200 import RenderConfig, ViewBatch, scenes
    wl = scenes.load("c3")
    V = a.views
    vb = ViewBatch(RenderConfig(), precision="fp64")
    st = torch.cuda.Stream()
    vb.set_stream(st.cuda_stream)
    vb.set_scene(wl.scene)
    vb.set_views(list(wl.cams)[:V])
    vb.render_ground_truth(wl.faces)
    ids = np.arange(V, dtype=np.int32)
    vb.set_timing(bool(a.timing))
    if a.bench_seq:
        for _ in range(a.n300):
            vb.zero_grads(); vb.step(ids, 300.0, 1.0 / V, write_maps=True); vb.finalize()
        if a.bench_seq & 2:
            vb.set_timing(True)
            vb.kernel_ms()
        if a.bench_seq & 4:
            vb.reset_stats()
        for _ in range(3):
            vb.zero_grads(); vb.step(ids, 300.0, 1.0 / V, write_maps=True); vb.finalize()
        torch.cuda.synchronize()
        if a.bench_seq & 2:
            print("kernel ms", vb.kernel_ms())
            vb.set_timing(False)
        if a.bench_seq & 8:
            print(vb.stats())
        a.n300 = 0
    for lam, reps in ((300.0, a.n300), (a.lam2, 2)):
        for r in range(reps):
            vb.zero_grads()
            vb.step(ids, lam, 1.0 / V, write_maps=True)
            vb.finalize()
            print(f"lambda {lam} rep {r} ok", flush=True)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
