"""Time the split iterations of the C4 loop piece by piece (maybe_split, the settled
step, the next deferred block), to locate the split-iteration cost.

  python scripts/c4_split_timing.py [--runs 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2412_03451_b200 import OptimConfig, Optimizer, Scene, scenes

    wl = scenes.load("c3")
    cams = list(wl.cams)[:512]
    out = []
    for r in range(a.runs):
        ocfg = OptimConfig(iterations=5000, views_per_step=8, split_grad_threshold=5e-5, seed=7)
        opt = Optimizer(Scene.empty(), cams, ocfg, precision="fp64")
        opt.render_ground_truth(wl.faces)
        opt.init_from_depth(5000, 7)
        opt.reset(0)
        torch.cuda.synchronize()
        rows = []
        for s in (1000, 2000, 3000, 4000):
            opt.run(s)  # up to the split iteration
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k = opt.maybe_split()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            opt.step()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            opt.run(s + 1 + 100)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            opt.run(s + 1 + 200)
            torch.cuda.synchronize()
            t4 = time.perf_counter()
            rows.append({"split_at": s, "split": k, "planes": opt.n_planes,
                         "maybe_split_ms": round((t1 - t0) * 1e3, 1), "step_ms": round((t2 - t1) * 1e3, 1),
                         "next100_ms": round((t3 - t2) * 1e3, 1), "then100_ms": round((t4 - t3) * 1e3, 1),
                         "replays": opt.stats().get("replays")})
        out.append(rows)
        opt.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
