"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU oracles.

``Oracle("ref")`` wraps oracle/_ref/libpsplat_ref.so (the reference's own C++
compiled through oracle/eigen_shim); ``Oracle("orc")`` wraps
oracle/_build/liboracle.so (the plain-C restatement, oracle/psplat_oracle.c).
Both expose the same calls with numpy in/out so tests can diff them directly.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
reference arm may import this module. The product (paper_2412_03451_b200) never
does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libpsplat_ref.so"),
    "orc": os.path.join(HERE, "_build", "liboracle.so"),
}


class Camera(C.Structure):
    """orc_camera: psplat::CameraView geometry (geometry.hpp:51-67)."""

    _fields_ = [
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("width", C.c_int32), ("height", C.c_int32),
        ("rot_wc", C.c_double * 9), ("t_wc", C.c_double * 3),
    ]

    def copy(self) -> "Camera":
        c = Camera()
        C.pointer(c)[0] = self
        return c


class Config(C.Structure):
    """orc_config: psplat::RenderConfig (renderer.hpp:10-21)."""

    _fields_ = [
        ("max_records", C.c_int32), ("normalize_by_alpha", C.c_int32),
        ("tile_size", C.c_int32), ("threads", C.c_int32),
        ("weight_floor", C.c_double), ("t_near", C.c_double), ("parallel_eps", C.c_double),
        ("alpha_floor", C.c_double), ("alpha1", C.c_double), ("alpha2", C.c_double),
    ]


@dataclass
class Planes:
    center: np.ndarray    # (n, 3) f64
    rotation: np.ndarray  # (n, 4) f64, (w, x, y, z)
    radii: np.ndarray     # (n, 4) f64, (x+, x-, y+, y-)
    ids: np.ndarray       # (n,) i64

    @property
    def n(self) -> int:
        return int(self.center.shape[0])

    @staticmethod
    def empty(n: int) -> "Planes":
        return Planes(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 4)),
                      np.arange(n, dtype=np.int64))

    def copy(self) -> "Planes":
        return Planes(self.center.copy(), self.rotation.copy(), self.radii.copy(), self.ids.copy())


def _p(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


_D, _F, _I32, _U16, _I64 = C.c_double, C.c_float, C.c_int32, C.c_uint16, C.c_int64


class Oracle:
    def __init__(self, which: str = "orc"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.p = which + "_"
        L, p = self.lib, self.p
        getattr(L, p + "lambda_schedule").restype = _D
        getattr(L, p + "lambda_schedule").argtypes = [C.c_int64, _D, _D, _D]
        getattr(L, p + "bin_primitives").restype = C.c_int64
        getattr(L, p + "fd_loss_gradient").restype = _D
        if which == "ref":
            L.ref_time_viewpass.restype = _D
            L.ref_init_from_depth.restype = C.c_int64

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    # ------------------------------------------------------------- config
    def default_config(self) -> Config:
        c = Config()
        self._f("default_config")(C.byref(c))
        return c

    def lambda_schedule(self, ite, base=20.0, rate=0.001, lmax=300.0) -> float:
        return self._f("lambda_schedule")(int(ite), base, rate, lmax)

    def plane_splat_weight(self, px, py, radii, lam):
        r = np.ascontiguousarray(radii, dtype=np.float64)
        out = np.zeros(11)
        self._f("plane_splat_weight")(_D(px), _D(py), _p(r, _D), _D(lam), _p(out, _D))
        return {"weight": out[0], "w_x": out[1], "w_y": out[2], "d_px": out[3],
                "d_py": out[4], "d_radii": out[5:9].copy(), "x_selected": bool(out[9])}

    # ------------------------------------------------------------- scenes
    def random_scene(self, seed: int, n: int) -> Planes:
        P = Planes.empty(n)
        self._f("random_scene")(C.c_uint64(seed), n, _p(P.center, _D), _p(P.rotation, _D),
                                _p(P.radii, _D), _p(P.ids, _I64))
        return P

    def make_view(self, w, h, focal, random_pose=False, seed=0) -> Camera:
        cam = Camera()
        self._f("make_view")(w, h, _D(focal), int(random_pose), C.c_uint64(seed), C.byref(cam))
        return cam

    def fill_random_targets(self, cam: Camera, seed: int):
        n = cam.width * cam.height
        td = np.zeros(n, np.float32)
        tn = np.zeros(3 * n, np.float32)
        self._f("fill_random_targets")(C.byref(cam), C.c_uint64(seed), _p(td, _F), _p(tn, _F))
        return td, tn

    # ------------------------------------------------------------- renderer
    def render_view(self, cam: Camera, P: Planes, lam: float, cfg: Config | None = None,
                    keep_records: bool = False):
        cfg = cfg or self.default_config()
        n = cam.width * cam.height
        M = cfg.max_records
        depth, normal, alpha = np.zeros(n), np.zeros(3 * n), np.zeros(n)
        rp = np.zeros(n * max(M, 1), np.int32) if keep_records else None
        rc = np.zeros(n, np.uint16) if keep_records else None
        st = self._f("render_view")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                    _p(P.rotation, _D), _p(P.radii, _D), _D(lam), C.byref(cfg),
                                    int(keep_records), _p(depth, _D), _p(normal, _D),
                                    _p(alpha, _D), _p(rp, _I32), _p(rc, _U16))
        if st != 0:
            raise ValueError(f"render_view: status {st}")
        out = {"depth": depth, "normal": normal, "alpha": alpha, "max_records": M}
        if keep_records:
            out["rec_prim"], out["rec_count"] = rp, rc
        return out

    def reference_render(self, cam: Camera, P: Planes, lam: float, cfg: Config | None = None):
        cfg = cfg or self.default_config()
        n = cam.width * cam.height
        depth, normal, alpha = np.zeros(n), np.zeros(3 * n), np.zeros(n)
        self._f("reference_render")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                    _p(P.rotation, _D), _p(P.radii, _D), _D(lam), C.byref(cfg),
                                    _p(depth, _D), _p(normal, _D), _p(alpha, _D))
        return {"depth": depth, "normal": normal, "alpha": alpha}

    def render_loss(self, cam: Camera, td, tn, maps, cfg: Config | None = None):
        cfg = cfg or self.default_config()
        n = cam.width * cam.height
        dd, dn, da = np.zeros(n), np.zeros(3 * n), np.zeros(n)
        loss = _D(0.0)
        st = self._f("render_loss")(C.byref(cam), _p(td, _F), _p(tn, _F), C.byref(cfg),
                                    _p(np.ascontiguousarray(maps["depth"]), _D),
                                    _p(np.ascontiguousarray(maps["normal"]), _D),
                                    _p(np.ascontiguousarray(maps["alpha"]), _D), C.byref(loss),
                                    _p(dd, _D), _p(dn, _D), _p(da, _D))
        if st != 0:
            raise ValueError(f"render_loss: status {st}")
        return {"loss": loss.value, "d_depth": dd, "d_normal": dn,
                "d_alpha": da if cfg.normalize_by_alpha else None}

    def backward(self, cam: Camera, P: Planes, lam: float, fwd, lg, cfg: Config | None = None,
                 grads: np.ndarray | None = None):
        cfg = cfg or self.default_config()
        g = np.zeros((P.n, 11)) if grads is None else grads
        err = C.create_string_buffer(256)
        da = lg.get("d_alpha")
        st = self._f("backward")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                 _p(P.rotation, _D), _p(P.radii, _D), _p(P.ids, _I64), _D(lam),
                                 C.byref(cfg), int(fwd["max_records"]),
                                 _p(fwd.get("rec_prim"), _I32), _p(fwd.get("rec_count"), _U16),
                                 _p(lg["d_depth"], _D), _p(lg["d_normal"], _D),
                                 _p(da, _D) if da is not None else None, _p(g, _D), err, 256)
        if st == 1:
            raise ValueError(err.value.decode())
        if st == 3:
            raise RuntimeError(err.value.decode())
        return g

    def bin_primitives(self, cam: Camera, P: Planes, lam: float, cfg: Config | None = None):
        cfg = cfg or self.default_config()
        ts = cfg.tile_size
        nt = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
        offs = np.zeros(nt + 1, np.int32)
        total = self._f("bin_primitives")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                          _p(P.rotation, _D), _p(P.radii, _D), _D(lam),
                                          C.byref(cfg), _p(offs, _I32), None, C.c_int64(0))
        items = np.zeros(max(total, 1), np.int32)
        self._f("bin_primitives")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                  _p(P.rotation, _D), _p(P.radii, _D), _D(lam), C.byref(cfg),
                                  _p(offs, _I32), _p(items, _I32), C.c_int64(total))
        return offs, items[:total]

    def gather_intersections(self, cam: Camera, P: Planes, lam: float, u: int, v: int,
                             cfg: Config | None = None):
        cfg = cfg or self.default_config()
        cap = max(P.n, 1)
        prim, z, w = np.zeros(cap, np.int32), np.zeros(cap), np.zeros(cap)
        cnt = self._f("gather_intersections")(C.byref(cam), C.c_int64(P.n), _p(P.center, _D),
                                              _p(P.rotation, _D), _p(P.radii, _D), _D(lam),
                                              C.byref(cfg), u, v, _p(prim, _I32), _p(z, _D),
                                              _p(w, _D), cap)
        return prim[:cnt], z[:cnt], w[:cnt]

    def fd_loss_gradient(self, cam, td, tn, P: Planes, prim, param, lam, step=1e-5,
                         cfg: Config | None = None) -> float:
        cfg = cfg or self.default_config()
        return self._f("fd_loss_gradient")(C.byref(cam), _p(td, _F), _p(tn, _F),
                                           C.c_int64(P.n), _p(P.center, _D), _p(P.rotation, _D),
                                           _p(P.radii, _D), C.c_int64(prim), int(param), _D(lam),
                                           _D(step), C.byref(cfg))

    # ------------------------------------------------------------- pipeline helpers
    def view_pass(self, cam, td, tn, P: Planes, lam, cfg: Config | None = None):
        """render_view(keep) + render_loss + backward, as Optimizer::step (optimizer.cpp:71-80)."""
        fwd = self.render_view(cam, P, lam, cfg, keep_records=True)
        lg = self.render_loss(cam, td, tn, fwd, cfg)
        g = self.backward(cam, P, lam, fwd, lg, cfg)
        return fwd, lg, g


class RefScenes:
    """The reference's synthetic generators (synthetic.cpp, scene_init.cpp) via _ref."""

    def __init__(self):
        self.o = Oracle("ref")
        self.lib = self.o.lib

    def room_faces(self, w, d, h, boxes, seed) -> np.ndarray:
        buf = np.zeros((64, 15))
        nf = self.lib.ref_room_faces(_D(w), _D(d), _D(h), boxes, C.c_uint64(seed),
                                     _p(buf, _D), 64)
        return buf[:nf].copy()

    def room_views(self, w, d, h, boxes, seed_room, n_views, seed_traj, width, height,
                   hfov_deg=75.0):
        cams = (Camera * n_views)()
        err = C.create_string_buffer(512)
        st = self.lib.ref_room_views(_D(w), _D(d), _D(h), boxes, C.c_uint64(seed_room), n_views,
                                     C.c_uint64(seed_traj), width, height, _D(hfov_deg), cams,
                                     err, 512)
        if st != 0:
            raise RuntimeError(err.value.decode())
        return cams

    def render_ground_truth(self, room, cams, threads=0):
        w, d, h, boxes, seed = room
        n = len(cams)
        npx = cams[0].width * cams[0].height
        td = np.zeros(n * npx, np.float32)
        tn = np.zeros(3 * n * npx, np.float32)
        self.lib.ref_render_ground_truth(_D(w), _D(d), _D(h), boxes, C.c_uint64(seed), n, cams,
                                         _p(td, _F), _p(tn, _F), threads)
        return td, tn

    def init_from_depth(self, cams, td, tn, n_prims, seed) -> Planes:
        P = Planes.empty(n_prims)
        got = self.lib.ref_init_from_depth(len(cams), cams, _p(td, _F), _p(tn, _F), n_prims,
                                           C.c_uint64(seed), _p(P.center, _D),
                                           _p(P.rotation, _D), _p(P.radii, _D), _p(P.ids, _I64))
        if got != n_prims:
            P = Planes(P.center[:got].copy(), P.rotation[:got].copy(), P.radii[:got].copy(),
                       P.ids[:got].copy())
        return P

    def time_viewpass(self, cam, td, tn, P: Planes, lam, threads, n_iter):
        cfg = self.o.default_config()
        cfg.threads = threads
        loss = _D(0.0)
        s = self.lib.ref_time_viewpass(C.byref(cam), _p(td, _F), _p(tn, _F), C.c_int64(P.n),
                                       _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
                                       _D(lam), C.byref(cfg), n_iter, C.byref(loss))
        return s, loss.value
