"""C4 loop timing in 100-iteration blocks, repeated, to locate run-to-run variance.

  python scripts/c4_variance.py [--runs 3] [--block 100] [--deterministic 0|1]
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
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--block", type=int, default=100)
    ap.add_argument("--iterations", type=int, default=5000)
    ap.add_argument("--deterministic", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_2412_03451_b200 import OptimConfig, Optimizer, Scene, scenes

    wl = scenes.load("c3")
    cams = list(wl.cams)[:512]
    out = []
    for r in range(a.runs):
        ocfg = OptimConfig(iterations=a.iterations, views_per_step=8, split_grad_threshold=5e-5, seed=7)
        opt = Optimizer(Scene.empty(), cams, ocfg, precision="fp64")
        opt.render_ground_truth(wl.faces)
        opt.init_from_depth(5000, 7)
        opt.reset(0)
        if a.deterministic:
            opt.set_deterministic(True)
        torch.cuda.synchronize()
        blocks = []
        rp = []
        t0 = time.perf_counter()
        it = 0
        while it < a.iterations:
            end = min(a.iterations, it + a.block)
            tb = time.perf_counter()
            rows = opt.run(end)
            blocks.append(round((time.perf_counter() - tb) * 1e3, 1))
            rp.append(opt.stats().get("replays"))
            it = end
        total = time.perf_counter() - t0
        out.append({"run": r, "seconds": round(total, 3), "planes": opt.n_planes, "block_ms": blocks, "replays_after_block": rp,
                    "stats": opt.stats() if hasattr(opt, "stats") else None})
        opt.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
