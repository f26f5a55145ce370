"""C4: the full optimisation loop on the device.

The room and trajectory of C3 (generate_box_room(6,5,3,4,7), sample_trajectory
seed 7), its first 512 views, 640x480, targets rendered on the device; planes from
init_from_depth(n=5000, seed=7) on the device (bit-identical to scene_init.cpp);
then Optimizer::run (maybe_split + step, Adam, renorm, clamp) for the given
iterations, and merge_planes at the end. Prints one JSON line.

  python scripts/run_c4.py [--iterations 5000] [--views-per-step 8] [--threshold 0.2]
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
    ap.add_argument("--iterations", type=int, default=5000)
    ap.add_argument("--views", type=int, default=512)
    ap.add_argument("--views-per-step", type=int, default=8)
    ap.add_argument("--planes", type=int, default=5000)
    ap.add_argument("--threshold", type=float, default=0.2, help="split_grad_threshold")
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--log-every", type=int, default=500)
    a = ap.parse_args()
    import torch
    from paper_2412_03451_b200 import OptimConfig, Optimizer, Scene, scenes

    wl = scenes.load("c3")
    cams = list(wl.cams)[:a.views]
    ocfg = OptimConfig(iterations=a.iterations, views_per_step=a.views_per_step,
                       split_grad_threshold=a.threshold, seed=7)
    opt = Optimizer(Scene.empty(), cams, ocfg, precision=a.precision)
    opt.render_ground_truth(wl.faces)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n0 = opt.init_from_depth(a.planes, 7)
    opt.reset(0)
    torch.cuda.synchronize()
    t_init = time.perf_counter() - t0

    log = []
    t0 = time.perf_counter()
    it = 0
    while it < a.iterations:
        # Optimizer::run in native code, in chunks of log_every iterations
        end = min(a.iterations, it + a.log_every)
        rows = opt.run(end)
        now = time.perf_counter()
        for r in (rows[0], rows[-1]):
            log.append({"iteration": r.iteration, "lambda": r.lam, "loss": r.loss,
                        "planes": r.primitive_count, "elapsed_s": now - t0})
        it = end
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t0
    t0 = time.perf_counter()
    inst = opt.merge_planes(opt.scene().center.mean(axis=0))
    t_merge = time.perf_counter() - t0
    print(json.dumps({
        "config": "C4: C3 room, %d views 640x480, %d -> %d planes, %d iterations, %d views/step, "
                  "split_grad_threshold %g, %s" % (a.views, n0, opt.n_planes, a.iterations,
                                                   a.views_per_step, a.threshold, a.precision),
        "init_from_depth_s": t_init, "run_s": t_run, "iterations_per_s": a.iterations / t_run,
        "view_passes_per_s": a.iterations * a.views_per_step / t_run,
        "merge_planes_s": t_merge, "instances": len(inst), "final_planes": opt.n_planes,
        "loss_first": log[0]["loss"], "loss_last": log[-1]["loss"], "log": log}))


if __name__ == "__main__":
    main()
