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

    # ------------------------------------------------------------- merge
    def merge_planes(self, P: Planes, scene_center=(0.0, 0.0, 0.0), normal_deg=25.0,
                     offset=0.1, adjacency=0.05, use_adjacency=True):
        """merge_planes (optimizer.cpp:236-299): instance index per primitive plus
        per-instance normal / offset / area, instances in the reference's order."""
        n = P.n
        inst = np.zeros(max(n, 1), np.int32)
        nrm, off, area = np.zeros((max(n, 1), 3)), np.zeros(max(n, 1)), np.zeros(max(n, 1))
        sc = np.ascontiguousarray(scene_center, np.float64)
        f = self._f("merge_planes")
        f.restype = C.c_int64
        k = f(C.c_int64(n), _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
              _p(P.ids, _I64), _p(sc, _D), _D(normal_deg), _D(offset), _D(adjacency),
              int(bool(use_adjacency)), _p(inst, _I32), _p(nrm, _D), _p(off, _D), _p(area, _D))
        return {"n": int(k), "instance_of": inst[:n], "normal": nrm[:k], "offset": off[:k],
                "area": area[:k]}

    def init_from_depth(self, cams, td, tn, n_prims, seed=0, radius_scale=0.5):
        """init_from_depth (scene_init.cpp:70-104) -> Planes (or the error code)."""
        P = Planes.empty(max(n_prims, 1))
        arr = (Camera * len(cams))(*cams)
        f = self.lib.ref_init_from_depth_cfg if self.p == "ref_" else self.lib.orc_init_from_depth
        f.restype = C.c_int64
        got = f(len(cams), arr, _p(np.ascontiguousarray(td, np.float32), _F),
                _p(np.ascontiguousarray(tn, np.float32), _F), int(n_prims), C.c_uint64(seed),
                _D(radius_scale), _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
                _p(P.ids, _I64))
        if got < 0:
            return int(got)
        return Planes(P.center[:got].copy(), P.rotation[:got].copy(), P.radii[:got].copy(),
                      P.ids[:got].copy())

    def rect_distance(self, ca, qa, ra, cb, qb, rb) -> float:
        f = self._f("rect_distance")
        f.restype = _D
        a = [np.ascontiguousarray(x, np.float64) for x in (ca, qa, ra, cb, qb, rb)]
        return f(*[_p(x, _D) for x in a])

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

    def time_render(self, cam, P: Planes, lam, threads, n_iter):
        """render_view(keep_records = false) n_iter times (BM_RenderView), seconds."""
        cfg = self.o.default_config()
        cfg.threads = threads
        f = self.lib.ref_time_render
        f.restype = _D
        return f(C.byref(cam), C.c_int64(P.n), _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
                 _D(lam), C.byref(cfg), n_iter)

    def time_viewpass(self, cam, td, tn, P: Planes, lam, threads, n_iter):
        cfg = self.o.default_config()
        cfg.threads = threads
        loss = _D(0.0)
        s = self.lib.ref_time_viewpass(C.byref(cam), _p(td, _F), _p(tn, _F), C.c_int64(P.n),
                                       _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
                                       _D(lam), C.byref(cfg), n_iter, C.byref(loss))
        return s, loss.value


# ---------------------------------------------------------------- optimiser
class OptimConfig(C.Structure):
    """orc_optim_config: psplat::OptimConfig (optimizer.hpp:10-27)."""

    _fields_ = [
        ("lr_center", C.c_double), ("lr_radii", C.c_double), ("lr_rotation", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
        ("split_interval", C.c_int64), ("split_grad_threshold", C.c_double),
        ("enable_split", C.c_int32), ("single_radii", C.c_int32),
        ("merge_normal_deg", C.c_double), ("merge_offset", C.c_double),
        ("merge_adjacency", C.c_double),
        ("merge_use_adjacency", C.c_int32), ("views_per_step", C.c_int32),
        ("seed", C.c_uint64), ("radii_floor", C.c_double),
    ]


@dataclass
class OptimState:
    """OptimState flattened (optimizer.hpp:63-70)."""
    planes: Planes
    m: np.ndarray        # (n, 11)
    v: np.ndarray        # (n, 11)
    step: np.ndarray     # (n,) i64
    rgs: np.ndarray      # (n, 4) radii_grad_sum
    rgc: np.ndarray      # (n,) i64 radii_grad_count
    iteration: int = 0
    next_id: int = 0

    @staticmethod
    def fresh(P: Planes, next_id: int | None = None) -> "OptimState":
        n = P.n
        return OptimState(P.copy(), np.zeros((n, 11)), np.zeros((n, 11)), np.zeros(n, np.int64),
                          np.zeros((n, 4)), np.zeros(n, np.int64), 0,
                          int(P.ids.max()) + 1 if next_id is None and n else (next_id or 0))


def _optim_lib(orc: "Oracle"):
    L = orc.lib
    if orc.p == "orc_":
        L.orc_view_for_slot.restype = C.c_int64
        L.orc_view_for_slot.argtypes = [C.c_uint64, C.c_int64, C.c_int64]
        L.orc_maybe_split.restype = C.c_int64
    else:
        L.ref_optimizer_create.restype = C.c_void_p
        L.ref_optimizer_create.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [
            C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
            C.c_double, C.c_double, C.c_double]
        L.ref_optimizer_destroy.argtypes = [C.c_void_p]
        L.ref_optimizer_step.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_optimizer_maybe_split.argtypes = [C.c_void_p]
        L.ref_optimizer_size.restype = C.c_int64
        L.ref_optimizer_size.argtypes = [C.c_void_p]
        L.ref_optimizer_view_for_slot.restype = C.c_int64
        L.ref_optimizer_view_for_slot.argtypes = [C.c_void_p, C.c_int64]
        L.ref_optimizer_get.argtypes = [C.c_void_p] + [C.c_void_p] * 11
        L.ref_optimizer_set_stats.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_optimizer_last_grads.argtypes = [C.c_void_p, C.c_void_p]
    return L


def default_optim_config(orc: "Oracle") -> OptimConfig:
    c = OptimConfig()
    getattr(orc.lib, orc.p + "default_optim_config")(C.byref(c))
    return c


class RestatedOptimizer:
    """Optimizer::step / maybe_split (optimizer.cpp:61-202) composed from the C
    restatement: orc render_view + render_loss + backward per view, then
    orc_accumulate_radii_grads and orc_apply_adam."""

    def __init__(self, orc: "Oracle", st: OptimState, cams, targets, ocfg: OptimConfig,
                 rcfg: Config | None = None, lam=(20.0, 0.001, 300.0)):
        assert orc.p == "orc_"
        self.o, self.L = orc, _optim_lib(orc)
        self.st, self.cams, self.targets, self.cfg = st, list(cams), list(targets), ocfg
        self.rcfg = rcfg or orc.default_config()
        self.lam = lam
        self.last_grads = None

    def view_for_slot(self, slot: int) -> int:
        return int(self.L.orc_view_for_slot(C.c_uint64(self.cfg.seed), len(self.cams), slot))

    def step(self) -> float:
        st, o = self.st, self.o
        lam = o.lambda_schedule(st.iteration, *self.lam)
        P = st.planes
        g = np.zeros((P.n, 11))
        V = int(self.cfg.views_per_step)
        scale = 1.0 / V
        loss = 0.0
        for k in range(V):
            vi = self.view_for_slot(st.iteration * V + k)
            cam, (td, tn) = self.cams[vi], self.targets[vi]
            f = o.render_view(cam, P, lam, self.rcfg, keep_records=True)
            lg = o.render_loss(cam, td, tn, f, self.rcfg)
            if V > 1:
                lg["loss"] *= scale
                for key in ("d_depth", "d_normal", "d_alpha"):
                    if lg.get(key) is not None:
                        lg[key] = lg[key] * scale
            loss += lg["loss"]
            o.backward(cam, P, lam, f, lg, self.rcfg, g)
        if not np.isfinite(loss):
            raise RuntimeError(f"optimizer: non-finite loss {loss}")
        self.last_grads = g.copy()
        self.L.orc_accumulate_radii_grads(C.c_int64(P.n), _p(g, _D), _p(st.rgs, _D), _p(st.rgc, _I64))
        self.L.orc_apply_adam(C.c_int64(P.n), _p(P.center, _D), _p(P.rotation, _D), _p(P.radii, _D),
                              _p(st.m, _D), _p(st.v, _D), _p(st.step, _I64), _p(g, _D),
                              C.byref(self.cfg))
        st.iteration += 1
        return loss

    def maybe_split(self) -> int:
        st = self.st
        n = st.planes.n
        out = OptimState.fresh(Planes.empty(2 * n))
        nid = C.c_int64(st.next_id)
        n_out = C.c_int64(0)
        P = st.planes
        k = self.L.orc_maybe_split(
            C.c_int64(n), C.c_int64(st.iteration), C.byref(self.cfg), _p(P.center, _D),
            _p(P.rotation, _D), _p(P.radii, _D), _p(P.ids, _I64), _p(st.m, _D), _p(st.v, _D),
            _p(st.step, _I64), _p(st.rgs, _D), _p(st.rgc, _I64), C.byref(nid),
            _p(out.planes.center, _D), _p(out.planes.rotation, _D), _p(out.planes.radii, _D),
            _p(out.planes.ids, _I64), _p(out.m, _D), _p(out.v, _D), _p(out.step, _I64),
            C.byref(n_out))
        if k < 0:
            return 0
        m = int(n_out.value)
        st.planes = Planes(out.planes.center[:m].copy(), out.planes.rotation[:m].copy(),
                           out.planes.radii[:m].copy(), out.planes.ids[:m].copy())
        st.m, st.v, st.step = out.m[:m].copy(), out.v[:m].copy(), out.step[:m].copy()
        st.rgs, st.rgc = np.zeros((m, 4)), np.zeros(m, np.int64)
        st.next_id = int(nid.value)
        return int(k)


class RefOptimizer:
    """The reference psplat::Optimizer, through its public API."""

    def __init__(self, ref: "Oracle", P: Planes, cams, targets, ocfg: OptimConfig,
                 rcfg: Config | None = None, lam=(20.0, 0.001, 300.0), next_id=None):
        assert ref.p == "ref_"
        self.L = _optim_lib(ref)
        rcfg = rcfg or ref.default_config()
        td = np.ascontiguousarray(np.concatenate([t[0] for t in targets]), np.float32)
        tn = np.ascontiguousarray(np.concatenate([t[1] for t in targets]), np.float32)
        cam_arr = (Camera * len(cams))(*cams)
        P = P.copy()
        self.h = self.L.ref_optimizer_create(
            P.n, P.center.ctypes.data, P.rotation.ctypes.data, P.radii.ctypes.data,
            P.ids.ctypes.data, int(P.ids.max()) + 1 if next_id is None else next_id, len(cams),
            C.cast(cam_arr, C.c_void_p), td.ctypes.data, tn.ctypes.data, C.addressof(ocfg),
            C.addressof(rcfg), *lam)
        self._keep = (td, tn, cam_arr, ocfg, rcfg)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_optimizer_destroy(self.h)
            self.h = None

    def step(self) -> float:
        loss = C.c_double(0)
        err = C.create_string_buffer(512)
        rc = self.L.ref_optimizer_step(self.h, C.byref(loss), err, 512)
        if rc == 1:
            raise RuntimeError(err.value.decode())
        if rc == 2:
            raise ValueError(err.value.decode())
        return loss.value

    def maybe_split(self) -> int:
        return int(self.L.ref_optimizer_maybe_split(self.h))

    def view_for_slot(self, slot: int) -> int:
        return int(self.L.ref_optimizer_view_for_slot(self.h, slot))

    def state(self) -> OptimState:
        n = int(self.L.ref_optimizer_size(self.h))
        s = OptimState.fresh(Planes.empty(n))
        it, nid = C.c_int64(0), C.c_int64(0)
        P = s.planes
        self.L.ref_optimizer_get(self.h, P.center.ctypes.data, P.rotation.ctypes.data,
                                 P.radii.ctypes.data, P.ids.ctypes.data, s.m.ctypes.data,
                                 s.v.ctypes.data, s.step.ctypes.data, s.rgs.ctypes.data,
                                 s.rgc.ctypes.data, C.byref(it), C.byref(nid))
        s.iteration, s.next_id = int(it.value), int(nid.value)
        return s

    def set_stats(self, iteration: int, rgs: np.ndarray, rgc: np.ndarray):
        rgs = np.ascontiguousarray(rgs, np.float64)
        rgc = np.ascontiguousarray(rgc, np.int64)
        self.L.ref_optimizer_set_stats(self.h, iteration, rgs.ctypes.data, rgc.ctypes.data)

    def last_grads(self) -> np.ndarray:
        n = int(self.L.ref_optimizer_size(self.h))
        g = np.zeros((n, 11))
        self.L.ref_optimizer_last_grads(self.h, g.ctypes.data)
        return g


class RefDataIO:
    """The reference's dataset I/O (dataio.cpp, compiled into oracle/_ref through the
    json/png test shims; oracle/ref_dataio.cpp)."""

    def __init__(self):
        self.lib = Oracle("ref").lib

    def _err(self, rc, err):
        if rc == 1:
            raise ValueError(err.value.decode())
        if rc:
            raise RuntimeError(err.value.decode())

    def write_map_f32(self, path, width, height, channels, data):
        err = C.create_string_buffer(512)
        a = np.ascontiguousarray(data, np.float32)
        self._err(self.lib.ref_write_map_f32(os.fsencode(path), width, height, channels, _p(a, _F), err, 512),
                  err)

    def read_map_f32(self, path, channels):
        err = C.create_string_buffer(512)
        w, h = C.c_int(0), C.c_int(0)
        self._err(self.lib.ref_read_map_f32(os.fsencode(path), channels, C.byref(w), C.byref(h), None,
                                            C.c_int64(0), err, 512), err)
        out = np.empty(w.value * h.value * channels, np.float32)
        self._err(self.lib.ref_read_map_f32(os.fsencode(path), channels, C.byref(w), C.byref(h), _p(out, _F),
                                            C.c_int64(out.size), err, 512), err)
        return w.value, h.value, out

    def write_dataset(self, root, cams, ids, td, tn, scene_center=(0.0, 0.0, 0.0), units="meters",
                      faces=None):
        err = C.create_string_buffer(512)
        arr = (Camera * len(cams))(*cams)
        ids = np.ascontiguousarray(ids, np.int32)
        sc = np.ascontiguousarray(scene_center, np.float64)
        fc = np.ascontiguousarray(faces if faces is not None else np.zeros((0, 15)), np.float64)
        self._err(self.lib.ref_write_dataset(os.fsencode(root), len(cams), arr, _p(ids, _I32),
                                             _p(np.ascontiguousarray(td, np.float32), _F),
                                             _p(np.ascontiguousarray(tn, np.float32), _F), _p(sc, _D),
                                             units.encode(), int(fc.shape[0]), _p(fc, _D), err, 512), err)

    def load_dataset(self, root, stride=1):
        """-> dict(cams, ids, td, tn, scene_center, units, has_meta, faces)."""
        err = C.create_string_buffer(512)
        nv, npx, nf = C.c_int(0), C.c_int64(0), C.c_int(0)
        f = self.lib.ref_load_dataset
        self._err(f(os.fsencode(root), int(stride), C.byref(nv), C.byref(npx), C.byref(nf), None, None, None,
                    None, None, None, 0, None, None, err, 512), err)
        cams = (Camera * max(nv.value, 1))()
        ids = np.empty(nv.value, np.int32)
        td, tn = np.empty(npx.value, np.float32), np.empty(3 * npx.value, np.float32)
        sc = np.zeros(3)
        units = C.create_string_buffer(64)
        has_meta = C.c_int(0)
        faces = np.zeros((max(nf.value, 1), 15))
        self._err(f(os.fsencode(root), int(stride), C.byref(nv), C.byref(npx), C.byref(nf), cams,
                    _p(ids, _I32), _p(td, _F), _p(tn, _F), _p(sc, _D), units, 64, C.byref(has_meta),
                    _p(faces, _D), err, 512), err)
        return {"cams": [cams[i] for i in range(nv.value)], "ids": ids, "td": td, "tn": tn,
                "scene_center": sc, "units": units.value.decode(), "has_meta": bool(has_meta.value),
                "faces": faces[:nf.value]}
