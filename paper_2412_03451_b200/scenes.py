"""Workload scenes of BASELINE.json (data/scenes/*.npz).

The files hold the plane sets, camera poses and synthetic room faces produced by
the reference's own generators (scripts/make_scenes.py). Targets are rendered on
the device from the faces (psg_render_ground_truth), so nothing here computes.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from ._lib import psg_camera
from .renderer import Scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENE_DIR = os.path.join(ROOT, "data", "scenes")

# SURVEY.md §8d names; c4 (split/merge loop) is not a fixed scene.
DESCRIPTIONS = {
    "c1": "synthetic box room (4x4x3, 0 boxes), 64 planes, 1 view 320x240",
    "c2": "synthetic room (4x4x3, 2 boxes), 2k planes, 32 views 640x480",
    "c2s": "synthetic room (4x4x3, 2 boxes), 2k planes, 32 views 320x240",
    "c3": "ScanNet-scale synthetic room (6x5x3, 4 boxes), 10k planes, 1024 views 640x480",
    "c5": "stress room (6x5x3, 4 boxes), 50k planes, 256 views 1296x968",
}


@dataclass
class Workload:
    name: str
    scene: Scene
    cams: "ctypes.Array"  # psg_camera[V]  # noqa: F821
    faces: np.ndarray     # (F, 15)
    room: np.ndarray
    target_checksum: np.ndarray

    @property
    def n_views(self) -> int:
        return len(self.cams)

    @property
    def width(self) -> int:
        return int(self.cams[0].width)

    @property
    def height(self) -> int:
        return int(self.cams[0].height)


def cams_from_array(a: np.ndarray):
    cams = (psg_camera * a.shape[0])()
    for i in range(a.shape[0]):
        c = cams[i]
        c.fx, c.fy, c.cx, c.cy = (float(x) for x in a[i, :4])
        c.width, c.height = int(a[i, 4]), int(a[i, 5])
        for k in range(9):
            c.rot_wc[k] = float(a[i, 6 + k])
        for k in range(3):
            c.t_wc[k] = float(a[i, 15 + k])
    return cams


def load(name: str) -> Workload:
    path = os.path.join(SCENE_DIR, f"{name}.npz")
    z = np.load(path)
    scene = Scene(z["center"], z["rotation"], z["radii"], z["ids"])
    return Workload(name, scene, cams_from_array(z["cams"]), z["faces"], z["room"],
                    z["target_checksum"])
