"""Host-side mirror of psplat::Optimizer (proj/core/include/psplat/optimizer.hpp)
with the whole step on the device.

  OptimConfig            optimizer.hpp:10-27
  SplatParams            splatting.hpp:8-13 (the lambda schedule)
  OptimState             optimizer.hpp:63-70 (scene + Adam + radii statistics)
  Optimizer.step         optimizer.cpp:61-98   -> psg_optim_step
  Optimizer.maybe_split  optimizer.cpp:142-202 -> psg_optim_maybe_split
  Optimizer.run          optimizer.cpp:204-214 (maybe_split + step loop)
  Optimizer.view_for_slot optimizer.cpp:49-59  -> psg_view_for_slot

Planes, Adam moments and the radii-gradient sums stay in HBM between steps; a
step reads back only the loss (8 bytes). With a communicator (comm_init) every
rank takes the slots k = rank mod N of each step and the gradients are summed
with one all-reduce before the identical Adam update on every rank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check
from .renderer import GradientBuffer, RenderConfig, Scene, ViewBatch, _ptr


@dataclass
class OptimConfig:
    iterations: int = 5000
    lr_center: float = 0.001
    lr_radii: float = 0.001
    lr_rotation: float = 0.001
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    split_interval: int = 1000
    split_grad_threshold: float = 0.2
    enable_split: bool = True
    single_radii: bool = False
    merge_normal_deg: float = 25.0  # merge_planes gates (optimizer.cpp:236-299)
    merge_offset: float = 0.1
    merge_adjacency: float = 0.05
    merge_use_adjacency: bool = True
    views_per_step: int = 1
    seed: int = 0
    radii_floor: float = 1e-4
    check_ranks: bool = False  # verify identical parameters across ranks each step


@dataclass
class SplatParams:
    lambda_base: float = 20.0
    lambda_rate: float = 0.001
    lambda_max: float = 300.0
    weight_floor: float = 1e-4


@dataclass
class OptimState:
    scene: Scene
    m: np.ndarray          # (n, 11)
    v: np.ndarray          # (n, 11)
    step: np.ndarray       # (n,) int64
    radii_grad_sum: np.ndarray    # (n, 4)
    radii_grad_count: np.ndarray  # (n,) int64
    iteration: int = 0
    next_id: int = 0


@dataclass
class PlaneInstance:
    """optimizer.hpp:48-56: a connected group of merged primitives."""
    member_ids: list
    member_indices: list
    normal: np.ndarray
    offset: float
    area: float
    id: int


@dataclass
class LossLogRow:
    iteration: int
    loss: float
    lam: float
    primitive_count: int


def view_for_slot(seed: int, n_views: int, slot: int) -> int:
    return int(_lib.lib().psg_view_for_slot(C.c_uint64(seed), n_views, slot))


class Optimizer(ViewBatch):
    """psplat::Optimizer with the step on the GPU (fp64 = the exact renderer)."""

    def __init__(self, scene: Scene, views, cfg: OptimConfig | None = None,
                 rcfg: RenderConfig | None = None, splat: SplatParams | None = None,
                 device: int = 0, precision: str = "fp64", next_id: int | None = None):
        super().__init__(rcfg, device, precision)
        self.ocfg = cfg or OptimConfig()
        self.splat = splat or SplatParams()
        self.set_scene(scene)
        views = list(views)
        if views and getattr(views[0], "target_depth", None) is not None:
            td = np.concatenate([np.asarray(v.target_depth, np.float32).ravel() for v in views])
            tn = np.concatenate([np.asarray(v.target_normal, np.float32).ravel() for v in views])
            self.set_views(views, td, tn)
        else:
            self.set_views(views)
        check(self.L.psg_optim_reset(self.h, 0, -1 if next_id is None else int(next_id)),
              "optim_reset")

    def reset(self, iteration: int = 0, next_id: int | None = None):
        """Fresh Adam state and radii statistics at `iteration` (lambda follows it)."""
        check(self.L.psg_optim_reset(self.h, int(iteration), -1 if next_id is None else int(next_id)),
              "optim_reset")

    def _c(self) -> _lib.psg_optim_config:
        o, s = self.ocfg, self.splat
        c = _lib.psg_optim_config()
        for f in ("lr_center", "lr_radii", "lr_rotation", "beta1", "beta2", "eps",
                  "split_grad_threshold", "radii_floor"):
            setattr(c, f, float(getattr(o, f)))
        c.split_interval = int(o.split_interval)
        c.enable_split = int(bool(o.enable_split))
        c.single_radii = int(bool(o.single_radii))
        c.views_per_step = int(o.views_per_step)
        c.check_ranks = int(bool(o.check_ranks))
        c.seed = int(o.seed) & ((1 << 64) - 1)
        c.lambda_base, c.lambda_rate, c.lambda_max = s.lambda_base, s.lambda_rate, s.lambda_max
        return c

    # ---- optimizer.hpp:82-98
    def step(self) -> float:
        loss = C.c_double(0.0)
        check(self.L.psg_optim_step(self.h, C.byref(self._c()), C.byref(loss)), "optim_step")
        return loss.value

    def step_local(self, rank: int, world: int):
        """This rank's share of the step (slots k mod world == rank) into the
        gradient buffer; all-reduce it (read_grads/set_grads or the device buffer),
        then step_finish()."""
        check(self.L.psg_optim_step_local(self.h, C.byref(self._c()), int(rank), int(world)),
              "optim_step_local")

    def step_finish(self) -> float:
        loss = C.c_double(0.0)
        check(self.L.psg_optim_step_finish(self.h, C.byref(self._c()), C.byref(loss)), "optim_step_finish")
        return loss.value

    def params_checksum(self) -> int:
        h = C.c_uint64(0)
        check(self.L.psg_params_checksum(self.h, C.byref(h)), "params_checksum")
        return h.value

    def apply(self):
        """optimizer.cpp:84-95 on the gradients already in the context."""
        check(self.L.psg_optim_apply(self.h, C.byref(self._c())), "optim_apply")

    def maybe_split(self) -> int:
        k = C.c_int64(0)
        check(self.L.psg_optim_maybe_split(self.h, C.byref(self._c()), C.byref(k)), "maybe_split")
        self.n_planes = int(self.L.psg_num_planes(self.h))
        return int(k.value)

    def run(self, iterations: int | None = None) -> list[LossLogRow]:
        """Optimizer::run (optimizer.cpp:204-214): the split + step loop runs in
        native code (psg_optim_run); returns its LossLogRow log."""
        end = self.ocfg.iterations if iterations is None else iterations
        start = self.iteration
        n = max(0, end - start)
        losses, lams = np.zeros(n), np.zeros(n)
        counts = np.zeros(n, np.int64)
        done = C.c_int64(0)
        rc = self.L.psg_optim_run(self.h, C.byref(self._c()), int(end), _ptr(losses), _ptr(lams),
                                  _ptr(counts), n, C.byref(done))
        self.n_planes = int(self.L.psg_num_planes(self.h))
        check(rc, "optim_run")
        k = int(done.value)
        return [LossLogRow(start + i, float(losses[i]), float(lams[i]), int(counts[i])) for i in range(k)]

    def lambda_at(self, ite: int) -> float:
        s = self.splat
        return float(self.L.psg_lambda_schedule(ite, s.lambda_base, s.lambda_rate, s.lambda_max))

    def view_for_slot(self, slot: int) -> int:
        return view_for_slot(self.ocfg.seed, self.n_views, slot)

    @property
    def iteration(self) -> int:
        it = C.c_int64(0)
        check(self.L.psg_optim_get_state(self.h, None, None, None, None, None, C.byref(it), None),
              "optim_get_state")
        return int(it.value)

    def scene(self) -> Scene:
        n = int(self.L.psg_num_planes(self.h))
        c, q, r = np.empty((n, 3)), np.empty((n, 4)), np.empty((n, 4))
        ids = np.empty(n, np.int64)
        check(self.L.psg_get_planes(self.h, _ptr(c), _ptr(q), _ptr(r), _ptr(ids)), "get_planes")
        return Scene(c, q, r, ids)

    def state(self) -> OptimState:
        sc = self.scene()
        n = sc.n
        m, v = np.empty((n, 11)), np.empty((n, 11))
        st, rgc = np.empty(n, np.int64), np.empty(n, np.int64)
        rgs = np.empty((n, 4))
        it, nid = C.c_int64(0), C.c_int64(0)
        check(self.L.psg_optim_get_state(self.h, _ptr(m), _ptr(v), _ptr(st), _ptr(rgs), _ptr(rgc),
                                         C.byref(it), C.byref(nid)), "optim_get_state")
        return OptimState(sc, m, v, st, rgs, rgc, int(it.value), int(nid.value))

    def load_state(self, s: OptimState):
        """Resume (Optimizer(OptimState, ...), optimizer.cpp:42-47)."""
        if s.m.shape[0] != s.scene.n:
            raise ValueError("optimizer state: adam/primitive size mismatch")
        self.set_scene(s.scene)
        f = lambda a, t: np.ascontiguousarray(a, t)  # noqa: E731
        check(self.L.psg_optim_set_state(self.h, _ptr(f(s.m, np.float64)), _ptr(f(s.v, np.float64)),
                                         _ptr(f(s.step, np.int64)),
                                         _ptr(f(s.radii_grad_sum, np.float64)),
                                         _ptr(f(s.radii_grad_count, np.int64)), int(s.iteration),
                                         int(s.next_id)), "optim_set_state")

    def merge_planes(self, scene_center=(0.0, 0.0, 0.0)) -> list[PlaneInstance]:
        """merge_planes(scene(), scene_center, cfg) (optimizer.cpp:236-299)."""
        o = self.ocfg
        n = int(self.L.psg_num_planes(self.h))
        inst = np.empty(max(n, 1), np.int32)
        nrm, off, area = np.empty((max(n, 1), 3)), np.empty(max(n, 1)), np.empty(max(n, 1))
        k = C.c_int64(0)
        sc = np.ascontiguousarray(scene_center, np.float64)
        check(self.L.psg_merge_planes(self.h, _ptr(sc), float(o.merge_normal_deg),
                                      float(o.merge_offset), float(o.merge_adjacency),
                                      int(bool(o.merge_use_adjacency)), _ptr(inst), _ptr(nrm),
                                      _ptr(off), _ptr(area), C.byref(k)), "merge_planes")
        ids = self.scene().ids
        out = []
        for t in range(int(k.value)):
            idx = np.nonzero(inst[:n] == t)[0].astype(np.int32)
            out.append(PlaneInstance(ids[idx].tolist(), idx.tolist(), nrm[t].copy(), float(off[t]),
                                     float(area[t]), t))
        return out

    def set_gradients(self, grads: np.ndarray, loss: float = 0.0):
        g = np.ascontiguousarray(grads, np.float64)
        check(self.L.psg_set_grads(self.h, _ptr(g), float(loss)), "set_grads")

    def last_gradients(self) -> GradientBuffer:
        g, _ = self.read_grads()
        gb = GradientBuffer(g.shape[0])
        gb.grads[:] = g
        return gb
