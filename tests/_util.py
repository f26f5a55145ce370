"""Test helpers: convert oracle-side fixtures into the product's API types."""
from __future__ import annotations

import numpy as np

from paper_2412_03451_b200 import CameraView, RenderConfig, Scene


def to_scene(P) -> Scene:
    return Scene(P.center.copy(), P.rotation.copy(), P.radii.copy(), P.ids.copy())


def to_view(cam, td=None, tn=None) -> CameraView:
    return CameraView(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                      np.array(list(cam.rot_wc)).reshape(3, 3), np.array(list(cam.t_wc)), td, tn)


def to_cfg(c) -> RenderConfig:
    return RenderConfig(max_records=c.max_records, weight_floor=c.weight_floor, t_near=c.t_near,
                        parallel_eps=c.parallel_eps, alpha_floor=c.alpha_floor,
                        normalize_by_alpha=bool(c.normalize_by_alpha), alpha1=c.alpha1,
                        alpha2=c.alpha2, tile_size=c.tile_size, threads=c.threads)


def bins_as_sets(offsets, items):
    return [frozenset(items[offsets[t]:offsets[t + 1]].tolist()) for t in range(len(offsets) - 1)]


def max_rel(a, b, floor=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))) \
        if a.size else 0.0
