"""init_from_depth on C3: the reference (oracle/_ref, CPU) vs the device path, on
the same targets (rendered bit-exactly on the device). Writes one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from oracle.oracle import Camera, Oracle
    from paper_2412_03451_b200 import ViewBatch, scenes
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    wl = scenes.load(name)
    vb = ViewBatch(precision="fp64")
    vb.set_views(list(wl.cams))
    vb.render_ground_truth(wl.faces)
    td = np.concatenate([vb.get_targets(k)[0] for k in range(wl.n_views)])
    tn = np.concatenate([vb.get_targets(k)[1] for k in range(wl.n_views)])
    cams = [Camera() for _ in range(wl.n_views)]
    for c, w in zip(cams, wl.cams):
        c.fx, c.fy, c.cx, c.cy, c.width, c.height = w.fx, w.fy, w.cx, w.cy, w.width, w.height
        for i in range(9):
            c.rot_wc[i] = w.rot_wc[i]
        for i in range(3):
            c.t_wc[i] = w.t_wc[i]
    ref = Oracle("ref")
    t0 = time.perf_counter()
    P = ref.init_from_depth(cams, td, tn, wl.scene.n, 7)
    t_ref = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vb.init_from_depth(wl.scene.n, 7)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    got = vb.planes()
    same = all(np.array_equal(a, b) for a, b in [(got.center, P.center), (got.rotation, P.rotation),
                                                 (got.radii, P.radii)])
    print(json.dumps({"config": name, "planes": int(P.n), "views": wl.n_views,
                      "reference_cpu_seconds": t_ref, "device_seconds": t_dev,
                      "speedup": t_ref / t_dev, "bitwise_equal": same,
                      "cpu": "reference init_from_depth is single-threaded (scene_init.cpp)"}))


if __name__ == "__main__":
    main()
