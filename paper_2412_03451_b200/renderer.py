"""Host-side mirror of the reference's psplat::Renderer operator API, over the C ABI.

Reference interface (proj/core/include/psplat/renderer.hpp):
  RenderConfig             renderer.hpp:10-21
  RenderedMaps             renderer.hpp:33-46
  ForwardResult            renderer.hpp:49-54
  GradientBuffer           renderer.hpp:62-66   (grads: (n, 11) = center 3, rotation 4, radii 4)
  LossGrads                renderer.hpp:68-73
  Renderer.render_view     renderer.hpp:98-99  / renderer.cpp:231-317
  Renderer.render_loss     renderer.hpp:104    / renderer.cpp:319-371
  Renderer.backward        renderer.hpp:108-110 / renderer.cpp:373-528
Scene / CameraView follow geometry.hpp:25-103 with numpy arrays.

Error behaviour matches the reference's exceptions: std::invalid_argument ->
ValueError, std::runtime_error ("backward: non-finite gradient for primitive id
N") -> RuntimeError. All arithmetic runs on the GPU; there is no CPU path.

``ViewBatch`` is the throughput API: views and targets live in HBM and one call
runs forward + L1 loss + backward for a list of views, exactly the inner loop of
Optimizer::step (optimizer.cpp:61-98).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, psg_camera, psg_render_config


@dataclass
class RenderConfig:
    max_records: int = 30
    weight_floor: float = 1e-4
    t_near: float = 0.01
    parallel_eps: float = 1e-8
    alpha_floor: float = 0.05
    normalize_by_alpha: bool = False
    alpha1: float = 5.0
    alpha2: float = 1.0
    tile_size: int = 16
    threads: int = 0  # accepted for API parity; the device ignores it

    def to_c(self) -> psg_render_config:
        c = psg_render_config()
        c.max_records = int(self.max_records)
        c.normalize_by_alpha = int(bool(self.normalize_by_alpha))
        c.tile_size = int(self.tile_size)
        c.threads = int(self.threads)
        c.weight_floor = float(self.weight_floor)
        c.t_near = float(self.t_near)
        c.parallel_eps = float(self.parallel_eps)
        c.alpha_floor = float(self.alpha_floor)
        c.alpha1 = float(self.alpha1)
        c.alpha2 = float(self.alpha2)
        return c


@dataclass
class Scene:
    """Scene::primitives as SoA: center (n,3), rotation (n,4) wxyz, radii (n,4), ids (n,)."""

    center: np.ndarray
    rotation: np.ndarray
    radii: np.ndarray
    ids: np.ndarray | None = None

    def __post_init__(self):
        self.center = np.ascontiguousarray(self.center, dtype=np.float64).reshape(-1, 3)
        self.rotation = np.ascontiguousarray(self.rotation, dtype=np.float64).reshape(-1, 4)
        self.radii = np.ascontiguousarray(self.radii, dtype=np.float64).reshape(-1, 4)
        n = self.center.shape[0]
        if self.rotation.shape[0] != n or self.radii.shape[0] != n:
            raise ValueError("Scene: center/rotation/radii length mismatch")
        if self.ids is None:
            self.ids = np.arange(n, dtype=np.int64)
        self.ids = np.ascontiguousarray(self.ids, dtype=np.int64)

    @property
    def n(self) -> int:
        return int(self.center.shape[0])

    @staticmethod
    def empty() -> "Scene":
        return Scene(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 4)))


@dataclass
class CameraView:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    rot_wc: np.ndarray = field(default_factory=lambda: np.eye(3))
    t_wc: np.ndarray = field(default_factory=lambda: np.zeros(3))
    target_depth: np.ndarray | None = None   # (H*W,) f32, <= 0 invalid
    target_normal: np.ndarray | None = None  # (H*W*3,) f32, 0-vector invalid
    id: int = 0

    def pixel_count(self) -> int:
        return int(self.width) * int(self.height)

    def to_c(self) -> psg_camera:
        c = psg_camera()
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        c.width, c.height = int(self.width), int(self.height)
        R = np.asarray(self.rot_wc, dtype=np.float64).reshape(9)
        t = np.asarray(self.t_wc, dtype=np.float64).reshape(3)
        for i in range(9):
            c.rot_wc[i] = R[i]
        for i in range(3):
            c.t_wc[i] = t[i]
        return c

    @staticmethod
    def from_c(c, target_depth=None, target_normal=None, id=0) -> "CameraView":
        return CameraView(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                          np.array(list(c.rot_wc), dtype=np.float64).reshape(3, 3),
                          np.array(list(c.t_wc), dtype=np.float64), target_depth, target_normal,
                          id)


@dataclass
class RenderedMaps:
    width: int
    height: int
    depth: np.ndarray   # (H*W,) f64
    normal: np.ndarray  # (H*W*3,) f64, camera frame, not renormalised
    alpha: np.ndarray   # (H*W,) f64


@dataclass
class ForwardResult:
    maps: RenderedMaps
    rec_prim: np.ndarray | None = None   # (H*W*M,) i32, -1 padded
    rec_count: np.ndarray | None = None  # (H*W,) u16
    max_records: int = 0


@dataclass
class LossGrads:
    loss: float
    d_depth: np.ndarray
    d_normal: np.ndarray
    d_alpha: np.ndarray | None = None


class GradientBuffer:
    """renderer.hpp:62-66; grads[i] = (d_center 3, d_rotation 4, d_radii 4)."""

    def __init__(self, n: int = 0):
        self.grads = np.zeros((n, 11), dtype=np.float64)

    def reset(self, n: int) -> None:
        self.grads = np.zeros((n, 11), dtype=np.float64)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a, n):
    a = np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
    if a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a


class _Context:
    """Owns one psg_context (one GPU)."""

    def __init__(self, device: int = 0, precision: str = "fp32"):
        self.L = _lib.lib()
        prec = {"fp32": _lib.PSG_FP32, "fp64": _lib.PSG_FP64, "mixed": _lib.PSG_MIXED}[precision]
        h = C.c_void_p()
        check(self.L.psg_create(int(device), prec, C.byref(h)), "psg_create")
        self.h = h
        self.device = device
        self.precision = precision
        self._scene_key = None

    def close(self):
        if getattr(self, "h", None):
            self.L.psg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_config(self, cfg: RenderConfig):
        c = cfg.to_c()
        check(self.L.psg_set_config(self.h, C.byref(c)), "set_config")

    def set_planes(self, scene: Scene):
        check(self.L.psg_set_planes(self.h, scene.n, _ptr(scene.center), _ptr(scene.rotation),
                                    _ptr(scene.radii), _ptr(scene.ids)), "set_planes")

    def set_stream(self, stream_ptr: int | None):
        check(self.L.psg_set_stream(self.h, C.c_void_p(stream_ptr or 0)), "set_stream")


class Renderer(_Context):
    """Drop-in for psplat::Renderer: same methods, arguments and exceptions."""

    def __init__(self, cfg: RenderConfig | None = None, device: int = 0, precision: str = "fp32"):
        super().__init__(device, precision)
        self.cfg = cfg or RenderConfig()

    def config(self) -> RenderConfig:
        return self.cfg

    def render_view(self, view: CameraView, scene: Scene, lam: float,
                    keep_records: bool = False) -> ForwardResult:
        if view.width < 1 or view.height < 1:
            raise ValueError("render_view: empty view")
        self.set_config(self.cfg)
        self.set_planes(scene)
        n = view.pixel_count()
        M = int(self.cfg.max_records)
        depth, normal, alpha = np.empty(n), np.empty(3 * n), np.empty(n)
        rp = np.empty(n * M, np.int32) if keep_records else None
        rc = np.empty(n, np.uint16) if keep_records else None
        cam = view.to_c()
        check(self.L.psg_render_view(self.h, C.byref(cam), float(lam), int(bool(keep_records)),
                                     _ptr(depth), _ptr(normal), _ptr(alpha), _ptr(rp), _ptr(rc)),
              "render_view")
        out = ForwardResult(RenderedMaps(view.width, view.height, depth, normal, alpha),
                            max_records=M)
        if keep_records:
            out.rec_prim, out.rec_count = rp, rc
        return out

    def render_loss(self, maps: RenderedMaps, view: CameraView) -> LossGrads:
        if maps.width != view.width or maps.height != view.height:
            raise ValueError("render_loss: resolution mismatch")  # renderer.cpp:320-321
        self.set_config(self.cfg)
        n = view.pixel_count()
        td = _f32(view.target_depth, n)
        tn = _f32(view.target_normal, 3 * n)
        depth = np.ascontiguousarray(maps.depth, dtype=np.float64)
        normal = np.ascontiguousarray(maps.normal, dtype=np.float64)
        alpha = np.ascontiguousarray(maps.alpha, dtype=np.float64)
        dd, dn = np.empty(n), np.empty(3 * n)
        da = np.empty(n) if self.cfg.normalize_by_alpha else None
        loss = C.c_double(0.0)
        cam = view.to_c()
        check(self.L.psg_render_loss(self.h, C.byref(cam), _ptr(td), _ptr(tn), _ptr(depth),
                                     _ptr(normal), _ptr(alpha), C.byref(loss), _ptr(dd), _ptr(dn),
                                     _ptr(da)), "render_loss")
        return LossGrads(loss.value, dd, dn, da)

    def backward(self, view: CameraView, scene: Scene, lam: float, fwd: ForwardResult,
                 loss_grads: LossGrads, gradbuf: GradientBuffer) -> None:
        if fwd.rec_count is None:
            raise ValueError("backward: forward pass ran without keep_records")
        self.set_config(self.cfg)
        self.set_planes(scene)
        if gradbuf.grads.shape != (scene.n, 11):
            gradbuf.reset(scene.n)  # renderer.cpp:503
        g = np.ascontiguousarray(gradbuf.grads, dtype=np.float64)
        rp = np.ascontiguousarray(fwd.rec_prim, dtype=np.int32)
        rc = np.ascontiguousarray(fwd.rec_count, dtype=np.uint16)
        dd = np.ascontiguousarray(loss_grads.d_depth, dtype=np.float64)
        dn = np.ascontiguousarray(loss_grads.d_normal, dtype=np.float64)
        da = (np.ascontiguousarray(loss_grads.d_alpha, dtype=np.float64)
              if loss_grads.d_alpha is not None and len(loss_grads.d_alpha) else None)
        bad = C.c_int64(-1)
        cam = view.to_c()
        st = self.L.psg_backward(self.h, C.byref(cam), float(lam), int(fwd.max_records), _ptr(rp),
                                 _ptr(rc), _ptr(dd), _ptr(dn), _ptr(da), _ptr(g), C.byref(bad))
        gradbuf.grads = g
        check(st, "backward")


class ViewBatch(_Context):
    """Resident views + fused forward/loss/backward over view lists (the hot path)."""

    # kernels of ours per psg_step + psg_finalize_grads: plane setup, rect/count,
    # crowded-tile list, capacity guard, scatter, record build (pairs, tiles),
    # persistent raster, crowded-tile raster (launched by every step: the crowded
    # tiles are counted on the device), loss fold, gradient finalise (CUB's scans not
    # counted)
    LAUNCHES_PER_STEP = 11

    def __init__(self, cfg: RenderConfig | None = None, device: int = 0, precision: str = "fp32"):
        super().__init__(device, precision)
        self.cfg = cfg or RenderConfig()
        self.set_config(self.cfg)
        self.n_views = 0
        self.n_planes = 0
        self._pinned = []

    def close(self):
        for p in getattr(self, "_pinned", []):
            self.L.psg_host_free(p)
        self._pinned = []
        super().close()

    def pinned(self, nbytes: int, dtype) -> np.ndarray:
        """Page-locked host buffer (freed with the context)."""
        p = self.L.psg_host_alloc(int(nbytes))
        if not p:
            raise MemoryError("psg_host_alloc failed")
        self._pinned.append(p)
        buf = (C.c_uint8 * int(nbytes)).from_address(p)
        return np.frombuffer(buf, dtype=dtype)

    def set_planes_host(self, center, rotation, radii, ids=None):
        n = int(np.asarray(center).size // 3)
        check(self.L.psg_set_planes(self.h, n, _ptr(center), _ptr(rotation), _ptr(radii),
                                    _ptr(None if ids is None else np.ascontiguousarray(ids, np.int64))),
              "set_planes")
        self.n_planes = n

    def read_grads_into(self, out: np.ndarray) -> float:
        loss = C.c_double(0.0)
        check(self.L.psg_read_grads(self.h, _ptr(out), C.byref(loss)), "read_grads")
        return loss.value

    def set_timing(self, enable: bool):
        check(self.L.psg_set_timing(self.h, int(bool(enable))), "set_timing")

    def kernel_ms(self) -> float:
        ms, n = C.c_double(0.0), C.c_int(0)
        check(self.L.psg_get_kernel_ms(self.h, C.byref(ms), C.byref(n)), "get_kernel_ms")
        return ms.value

    def launches_per_step(self, crowded: bool = True) -> int:
        # a synchronous (deterministic) step launches the crowded-tile kernel only when
        # there are crowded tiles; the default step always does
        return self.LAUNCHES_PER_STEP - (0 if crowded or not self._deterministic else 1)

    def set_scene(self, scene: Scene):
        self.set_planes(scene)
        self.n_planes = scene.n

    def set_views(self, cams, target_depth=None, target_normal=None):
        """cams: sequence of psg_camera or CameraView; targets concatenated in view order."""
        arr = (psg_camera * len(cams))()
        for i, c in enumerate(cams):
            arr[i] = c.to_c() if isinstance(c, CameraView) else c
        td = None if target_depth is None else np.ascontiguousarray(target_depth, np.float32)
        tn = None if target_normal is None else np.ascontiguousarray(target_normal, np.float32)
        check(self.L.psg_set_views(self.h, len(cams), arr, _ptr(td), _ptr(tn)), "set_views")
        self.n_views = len(cams)
        self._cams = arr

    def load_dataset(self, ds, chunk_views: int = 64, threads: int = 0):
        """Register a PSMP dataset's views and stream its targets into HBM
        (psg_load_dataset: reader threads into pinned staging, overlapped copies)."""
        check(self.L.psg_load_dataset(self.h, ds.h, int(chunk_views), int(threads)), "load_dataset")
        self.n_views = ds.n_views
        self._cams = ds._cams

    def init_from_depth(self, n_primitives: int, seed: int = 0, radius_scale: float = 0.5) -> int:
        """init_from_depth (scene_init.cpp:70-104) from the resident targets; the
        context's planes are replaced. Returns the primitive count."""
        n = C.c_int64(0)
        check(self.L.psg_init_from_depth(self.h, int(n_primitives), C.c_uint64(seed), float(radius_scale),
                                         C.byref(n)), "init_from_depth")
        self.n_planes = n.value
        return n.value

    def planes(self) -> Scene:
        """The context's current planes (psg_get_planes)."""
        n = int(self.L.psg_num_planes(self.h))
        c, q, r = np.empty((n, 3)), np.empty((n, 4)), np.empty((n, 4))
        ids = np.empty(n, np.int64)
        check(self.L.psg_get_planes(self.h, _ptr(c), _ptr(q), _ptr(r), _ptr(ids)), "get_planes")
        return Scene(c, q, r, ids)

    def render_ground_truth(self, faces: np.ndarray):
        f = np.ascontiguousarray(faces, dtype=np.float64).reshape(-1, 15)
        check(self.L.psg_render_ground_truth(self.h, f.shape[0], _ptr(f)), "render_ground_truth")

    def _range_pixels(self, first: int, count: int) -> int:
        if first < 0 or count < 0 or first + count > len(self._cams):
            raise ValueError("bad view range")
        return sum(self._cams[i].width * self._cams[i].height for i in range(first, first + count))

    def update_targets(self, first: int, count: int, td: np.ndarray, tn: np.ndarray):
        npx = self._range_pixels(first, count)
        td, tn = _f32(td, npx), _f32(tn, 3 * npx)  # contiguous f32 (pinned buffers pass as they are)
        check(self.L.psg_update_targets(self.h, first, count, _ptr(td), _ptr(tn)), "update_targets")

    def get_targets(self, view: int):
        c = self._cams[view]
        n = c.width * c.height
        td, tn = np.empty(n, np.float32), np.empty(3 * n, np.float32)
        check(self.L.psg_get_targets(self.h, view, _ptr(td), _ptr(tn)), "get_targets")
        return td, tn

    _deterministic = False

    def set_deterministic(self, enable: bool = True):
        """Bitwise run-to-run reproducible gradients and loss (fixed-order reductions)."""
        check(self.L.psg_set_deterministic(self.h, int(bool(enable))), "set_deterministic")
        self._deterministic = bool(enable)

    def zero_grads(self):
        check(self.L.psg_zero_grads(self.h), "zero_grads")

    def step(self, view_ids, lam: float, view_scale: float = 1.0, write_maps: bool = False,
             backward: bool = True):
        ids = np.ascontiguousarray(view_ids, dtype=np.int32)
        flags = (_lib.PSG_STEP_WRITE_MAPS if write_maps else 0) | \
                (0 if backward else _lib.PSG_STEP_NO_BACKWARD)
        check(self.L.psg_step(self.h, _ptr(ids), int(ids.size), float(lam), float(view_scale),
                              flags), "step")

    def step_host(self, first: int, count: int, lam: float, target_depth, target_normal,
                  view_scale: float = 1.0, chunk_views: int = 128, backward: bool = True,
                  write_maps: bool = False):
        """Fused step over views [first, first+count) with their targets copied from
        host memory, chunked so the copies overlap the compute (psg_step_host)."""
        flags = (0 if backward else _lib.PSG_STEP_NO_BACKWARD) | \
                (_lib.PSG_STEP_WRITE_MAPS if write_maps else 0)
        npx = self._range_pixels(first, count)
        target_depth, target_normal = _f32(target_depth, npx), _f32(target_normal, 3 * npx)
        check(self.L.psg_step_host(self.h, int(first), int(count), float(lam), float(view_scale),
                                   flags, _ptr(target_depth), _ptr(target_normal),
                                   int(chunk_views)), "step_host")

    def finalize(self):
        bad = C.c_int64(-1)
        check(self.L.psg_finalize_grads(self.h, C.byref(bad)), "finalize_grads")

    def read_grads(self):
        g = np.empty((self.n_planes, 11))
        loss = C.c_double(0.0)
        check(self.L.psg_read_grads(self.h, _ptr(g), C.byref(loss)), "read_grads")
        return g, loss.value

    def view_losses(self, n: int) -> np.ndarray:
        out = np.empty(n)
        check(self.L.psg_read_view_losses(self.h, _ptr(out), n), "read_view_losses")
        return out

    def read_step_maps(self, k: int, width: int, height: int):
        n = width * height
        d, nn, a = np.empty(n, np.float32), np.empty(3 * n, np.float32), np.empty(n, np.float32)
        check(self.L.psg_read_step_maps(self.h, k, _ptr(d), _ptr(nn), _ptr(a)), "read_step_maps")
        return d, nn, a

    def stats(self) -> dict:
        s = _lib.psg_stats()
        check(self.L.psg_get_stats(self.h, C.byref(s)), "get_stats")
        return {f: getattr(s, f) for f, _ in s._fields_}

    def set_pair_limit(self, limit: int):
        """Largest bin-entry count of one binning pass (<= 2^31 - 1); larger steps are
        split into view groups (psg_set_pair_limit)."""
        check(self.L.psg_set_pair_limit(self.h, int(limit)), "set_pair_limit")

    def reset_stats(self):
        check(self.L.psg_reset_stats(self.h), "reset_stats")

    def stream(self) -> int:
        return int(self.L.psg_get_stream(self.h) or 0)

    # ---- multi-GPU
    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, _lib.PSG_NCCL_ID_BYTES)
        check(self.L.psg_comm_init(self.h, buf, nranks, rank), "comm_init")

    def allreduce_grads(self):
        check(self.L.psg_allreduce_grads(self.h), "allreduce_grads")


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(_lib.PSG_NCCL_ID_BYTES)
    check(_lib.lib().psg_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


def lambda_schedule(ite: int, base: float = 20.0, rate: float = 0.001, lmax: float = 300.0):
    """splatting.cpp:7-10."""
    return _lib.lib().psg_lambda_schedule(int(ite), base, rate, lmax)
