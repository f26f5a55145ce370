"""Small workload covering every kernel path, for compute-sanitizer runs:
persistent resident kernel (fused + forward-with-records), crowded-tile launch
(sorted streaming and unsorted), drop-in loss and backward, GT render, the
host-staged step, deterministic reductions, init_from_depth, the device
optimiser (Adam, split) and merge_planes.

  compute-sanitizer --tool memcheck python scripts/sanitize_case.py
  compute-sanitizer --tool racecheck python scripts/sanitize_case.py --small
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from _util import to_scene, to_view  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2412_03451_b200 import GradientBuffer, Renderer, ViewBatch, scenes  # noqa: E402


def main():
    small = "--small" in sys.argv
    orc = Oracle("orc")
    for prec in ("fp64", "mixed", "fp32"):
        for n_planes in ((24, 400) if small else (24, 400, 1500)):
            P = orc.random_scene(5, n_planes)
            cam = orc.make_view(40, 24, 20.0, True, 5)
            td, tn = orc.fill_random_targets(cam, 5)
            r = Renderer(precision=prec)
            v = to_view(cam, td, tn)
            f = r.render_view(v, to_scene(P), 30.0, keep_records=True)
            lg = r.render_loss(f.maps, v)
            gb = GradientBuffer(P.n)
            r.backward(v, to_scene(P), 30.0, f, lg, gb)
            vb = ViewBatch(precision=prec)
            vb.set_scene(to_scene(P))
            vb.set_views([v], td, tn)
            vb.zero_grads()
            vb.step([0], 30.0, 1.0, write_maps=True)
            vb.finalize()
            vb.read_grads()
    wl = scenes.load("c1")
    vb = ViewBatch(precision="fp64")
    vb.set_scene(wl.scene)
    vb.set_views(list(wl.cams)[:2])
    vb.render_ground_truth(wl.faces)
    vb.zero_grads()
    vb.step([0, 1], 300.0, 0.5)
    vb.finalize()
    g0 = vb.read_grads()[0]
    # host-staged step and the deterministic reductions
    td = np.concatenate([vb.get_targets(i)[0] for i in range(2)])
    tn = np.concatenate([vb.get_targets(i)[1] for i in range(2)])
    vb.zero_grads()
    vb.step_host(0, 2, 300.0, td, tn, 0.5, chunk_views=1)
    vb.set_deterministic(True)
    vb.zero_grads()
    vb.step([0, 1], 20.0, 0.5)
    vb.finalize()
    # init_from_depth, device Optimizer (Adam + split) and merge_planes
    from paper_2412_03451_b200 import OptimConfig, Optimizer, Scene
    opt = Optimizer(Scene.empty(), list(wl.cams)[:2],
                    OptimConfig(iterations=6, views_per_step=2, split_interval=3,
                                split_grad_threshold=0.0, seed=3))
    opt.render_ground_truth(wl.faces)
    opt.init_from_depth(200, 7)
    opt.reset(0)
    while opt.iteration < 6:
        opt.maybe_split()
        opt.step()
    inst = opt.merge_planes((0.0, 0.0, 0.0))
    print("sanitize_case: ok", np.isfinite(g0).all(), opt.n_planes, len(inst))


if __name__ == "__main__":
    main()
