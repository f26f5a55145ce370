"""Generate the BASELINE.json workload scenes with the reference's own generators.

Runs the reference's generate_box_room / sample_trajectory / render_ground_truth /
init_from_depth (proj/core/src/synthetic.cpp, scene_init.cpp), compiled into
oracle/_ref/libpsplat_ref.so, and stores the plane sets, camera poses and room
faces under data/scenes/<name>.npz. Targets are not stored: they are re-rendered
exactly from the faces (on the device by psg_render_ground_truth, or on the CPU
by the reference's render_ground_truth) wherever they are needed.

Configs (seed 7, hfov 75 deg, targets from render_ground_truth):
  c1: room(4,4,3,0), 100-view trajectory (view 0 used), 320x240, init n=64
  c2: room(4,4,3,2), 32 views, 640x480, init n=2000. sample_trajectory throws for
      fewer than 48 views on this 16-face room (coverage, synthetic.cpp:285-299), so
      a 48-view trajectory is sampled and its first 32 views are used.
  c2s: c2 at 320x240 (the shape of the reference's BM_ForwardBackward,
      benchmarks/render_bench.cpp:54-67, whose own 8-pose BenchScene cannot pass
      sample_trajectory's coverage check on this room)
  c3: room(6,5,3,4), 1024 views, 640x480, init n=10000
  c5: room(6,5,3,4), 256 views, 1296x968, init n=50000

Usage: python scripts/make_scenes.py [c1 c2 c3 c5]
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Camera, RefScenes  # noqa: E402

CONFIGS = {
    "c1": dict(room=(4.0, 4.0, 3.0, 0, 7), n_views=100, W=320, H=240, n_planes=64),
    "c2": dict(room=(4.0, 4.0, 3.0, 2, 7), n_views=32, traj_views=48, W=640, H=480,
               n_planes=2000),
    "c2s": dict(room=(4.0, 4.0, 3.0, 2, 7), n_views=32, traj_views=48, W=320, H=240,
                n_planes=2000),
    "c3": dict(room=(6.0, 5.0, 3.0, 4, 7), n_views=1024, W=640, H=480, n_planes=10000),
    "c5": dict(room=(6.0, 5.0, 3.0, 4, 7), n_views=256, W=1296, H=968, n_planes=50000),
}


def cams_to_array(cams) -> np.ndarray:
    """(V, 17) f64: fx, fy, cx, cy, W, H, rot_wc[9] row-major, t_wc... -> see CAM_COLS."""
    out = np.zeros((len(cams), 20))
    for i, c in enumerate(cams):
        out[i, :4] = (c.fx, c.fy, c.cx, c.cy)
        out[i, 4:6] = (c.width, c.height)
        out[i, 6:15] = list(c.rot_wc)
        out[i, 15:18] = list(c.t_wc)
    return out


def array_to_cams(a: np.ndarray):
    cams = (Camera * a.shape[0])()
    for i in range(a.shape[0]):
        c = cams[i]
        c.fx, c.fy, c.cx, c.cy = a[i, :4]
        c.width, c.height = int(a[i, 4]), int(a[i, 5])
        for k in range(9):
            c.rot_wc[k] = a[i, 6 + k]
        for k in range(3):
            c.t_wc[k] = a[i, 15 + k]
    return cams


def make(name: str) -> str:
    cfg = CONFIGS[name]
    rs = RefScenes()
    w, d, h, boxes, seed = cfg["room"]
    t0 = time.time()
    faces = rs.room_faces(w, d, h, boxes, seed)
    cams = rs.room_views(w, d, h, boxes, seed, cfg.get("traj_views", cfg["n_views"]), seed,
                         cfg["W"], cfg["H"], 75.0)
    cams = (Camera * cfg["n_views"])(*cams[: cfg["n_views"]])
    t1 = time.time()
    td, tn = rs.render_ground_truth(cfg["room"], cams, threads=0)
    t2 = time.time()
    planes = rs.init_from_depth(cams, td, tn, cfg["n_planes"], seed)
    t3 = time.time()
    out = os.path.join(ROOT, "data", "scenes", f"{name}.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(
        out, room=np.array([w, d, h, boxes, seed], dtype=np.float64), faces=faces,
        cams=cams_to_array(cams), center=planes.center, rotation=planes.rotation,
        radii=planes.radii, ids=planes.ids,
        target_checksum=np.array([float(np.sum(td, dtype=np.float64)),
                                  float(np.sum(tn, dtype=np.float64))]))
    print(f"{name}: {len(faces)} faces, {len(cams)} views {cfg['W']}x{cfg['H']}, "
          f"{planes.n} planes; trajectory {t1 - t0:.1f}s, GT {t2 - t1:.1f}s, init {t3 - t2:.1f}s "
          f"-> {out}")
    return out


if __name__ == "__main__":
    for nm in (sys.argv[1:] or ["c1", "c2", "c3"]):
        make(nm)
