"""PSMP dataset I/O (reference proj/core/include/psplat/dataio.hpp, dataio.cpp).

  write_map_f32 / read_map_f32   dataio.cpp:65-97   (C ABI)
  Dataset (load_dataset)         dataio.cpp:136-201 (C ABI: psg_dataset_*; meta.json here)
  write_dataset                  dataio.cpp:203-248 (writer for fixtures and exports)

Errors keep the reference's types: std::runtime_error (bad files, with the path in
the message) -> RuntimeError, std::invalid_argument (stride < 1) -> ValueError.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, psg_camera
from .renderer import CameraView, _ptr


def write_map_f32(path: str, width: int, height: int, channels: int, data: np.ndarray) -> None:
    a = np.ascontiguousarray(data, np.float32).reshape(-1)
    if a.size != width * height * channels:
        raise ValueError("write_map_f32: data size does not match width*height*channels")
    check(_lib.lib().psg_write_map_f32(os.fsencode(path), width, height, channels, _ptr(a)),
          "write_map_f32")


def read_map_f32(path: str, expected_channels: int):
    """Returns (width, height, data[h*w*channels] f32)."""
    L = _lib.lib()
    w, h = C.c_int(0), C.c_int(0)
    check(L.psg_read_map_f32(os.fsencode(path), expected_channels, C.byref(w), C.byref(h), None, 0),
          "read_map_f32")
    out = np.empty(w.value * h.value * expected_channels, np.float32)
    check(L.psg_read_map_f32(os.fsencode(path), expected_channels, C.byref(w), C.byref(h), _ptr(out),
                             out.size), "read_map_f32")
    return w.value, h.value, out


@dataclass
class GtFace:
    """synthetic.hpp GtFace as stored in meta.json (dataio.cpp:186-196)."""
    instance_id: int
    center: np.ndarray
    u_axis: np.ndarray
    v_axis: np.ndarray
    half_u: float
    half_v: float

    @property
    def normal(self) -> np.ndarray:
        return np.cross(self.u_axis, self.v_axis)


@dataclass
class SceneMeta:
    scene_center: np.ndarray = field(default_factory=lambda: np.zeros(3))
    units: str = "meters"
    gt_faces: list = field(default_factory=list)


class Dataset:
    """load_dataset(root, stride): cameras parsed and every map header checked on
    open; targets are read (and validated) by the library's reader threads."""

    def __init__(self, root: str, stride: int = 1):
        self.L = _lib.lib()
        self.root = root
        h = C.c_void_p()
        check(self.L.psg_dataset_open(os.fsencode(root), int(stride), C.byref(h)), "load_dataset")
        self.h = h
        n, npx = C.c_int(0), C.c_int64(0)
        check(self.L.psg_dataset_size(self.h, C.byref(n), C.byref(npx)), "dataset_size")
        self.n_views, self.n_pixels = n.value, npx.value
        self._cams = (psg_camera * max(self.n_views, 1))()
        self.ids = np.empty(self.n_views, np.int32)
        check(self.L.psg_dataset_cameras(self.h, self._cams, _ptr(self.ids)), "dataset_cameras")
        self.meta, self.has_meta = SceneMeta(), False
        mp = os.path.join(root, "meta.json")
        if os.path.exists(mp):  # dataio.cpp:174-199
            try:
                with open(mp) as f:
                    j = json.load(f)
            except ValueError as e:
                raise RuntimeError(f"{mp}: {e}") from e
            self.meta.scene_center = np.asarray(j["scene_center"], np.float64)
            self.meta.units = j.get("units", "meters")
            for fj in j.get("gt_faces", []):
                self.meta.gt_faces.append(GtFace(int(fj["id"]), np.asarray(fj["center"], float),
                                                 np.asarray(fj["u_axis"], float),
                                                 np.asarray(fj["v_axis"], float),
                                                 float(fj["half_u"]), float(fj["half_v"])))
            self.has_meta = True

    def close(self):
        if getattr(self, "h", None):
            self.L.psg_dataset_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def cameras(self) -> list:
        return [self._cams[i] for i in range(self.n_views)]

    def read(self, first: int = 0, count: int | None = None, threads: int = 0):
        """Targets of views [first, first+count), concatenated: (depth, normal) f32."""
        count = self.n_views - first if count is None else count
        c = self._cams
        npx = sum(c[i].width * c[i].height for i in range(first, first + count))
        td, tn = np.empty(npx, np.float32), np.empty(3 * npx, np.float32)
        check(self.L.psg_dataset_read(self.h, first, count, _ptr(td), _ptr(tn), int(threads)),
              "dataset_read")
        return td, tn

    def views(self, threads: int = 0) -> list:
        """CameraView list with targets, as load_dataset returns it."""
        td, tn = self.read(threads=threads)
        out, o = [], 0
        for i in range(self.n_views):
            c = self._cams[i]
            n = c.width * c.height
            out.append(CameraView.from_c(c, td[o:o + n].copy(), tn[3 * o:3 * (o + n)].copy(),
                                         int(self.ids[i])))
            o += n
        return out


def write_dataset(root: str, views, meta: SceneMeta | None = None) -> None:
    """write_dataset (dataio.cpp:203-248): cameras.txt at 17 significant digits,
    depth/ and normal/ PSMP maps, meta.json."""
    meta = meta or SceneMeta()
    os.makedirs(os.path.join(root, "depth"), exist_ok=True)
    os.makedirs(os.path.join(root, "normal"), exist_ok=True)
    with open(os.path.join(root, "cameras.txt"), "w") as f:
        for v in views:
            R = np.asarray(v.rot_wc, np.float64).reshape(3, 3)
            t = np.asarray(v.t_wc, np.float64).reshape(3)
            m = np.zeros(16)
            m[[0, 1, 2, 4, 5, 6, 8, 9, 10]] = R.reshape(-1)
            m[[3, 7, 11]] = t
            m[15] = 1.0
            vals = [v.fx, v.fy, v.cx, v.cy]
            f.write(f"{int(v.id)} " + " ".join("%.17g" % x for x in vals) +
                    f" {int(v.width)} {int(v.height)} " + " ".join("%.17g" % x for x in m) + "\n")
            write_map_f32(os.path.join(root, "depth", f"{int(v.id)}.f32"), v.width, v.height, 1,
                          v.target_depth)
            write_map_f32(os.path.join(root, "normal", f"{int(v.id)}.f32"), v.width, v.height, 3,
                          v.target_normal)
    j = {"scene_center": [float(x) for x in np.asarray(meta.scene_center).reshape(3)],
         "units": meta.units}
    if meta.gt_faces:
        j["gt_faces"] = [{"id": f.instance_id, "center": list(map(float, f.center)),
                          "u_axis": list(map(float, f.u_axis)), "v_axis": list(map(float, f.v_axis)),
                          "half_u": f.half_u, "half_v": f.half_v} for f in meta.gt_faces]
    # nlohmann::json objects are std::map-ordered: the reference writes keys sorted
    with open(os.path.join(root, "meta.json"), "w") as f:
        f.write(json.dumps(j, indent=2, sort_keys=True) + "\n")


# ---- PSCK checkpoints of the optimiser state (dataio.cpp:250-330) ----------
_CK_MAGIC, _CK_VERSION = b"PSCK", 1
_CK_REC = np.dtype([("id", "<i8"), ("center", "<f8", 3), ("rotation", "<f8", 4), ("radii", "<f8", 4),
                    ("step", "<i8"), ("m", "<f8", 11), ("v", "<f8", 11), ("rgs", "<f8", 4),
                    ("rgc", "<i8")])


def save_checkpoint(path: str, state, config_hash: int) -> None:
    """save_checkpoint: magic, version, config hash, iteration, next id, count,
    then per primitive id, centre, rotation, radii, Adam step/m/v, radii sums."""
    sc = state.scene
    n = sc.n
    rec = np.zeros(n, _CK_REC)
    rec["id"], rec["center"], rec["rotation"], rec["radii"] = sc.ids, sc.center, sc.rotation, sc.radii
    rec["step"], rec["m"], rec["v"] = state.step, state.m, state.v
    rec["rgs"], rec["rgc"] = state.radii_grad_sum, state.radii_grad_count
    hdr = _CK_MAGIC + np.array([_CK_VERSION], "<u4").tobytes() + \
        np.array([config_hash & ((1 << 64) - 1)], "<u8").tobytes() + \
        np.array([state.iteration, state.next_id], "<i8").tobytes() + np.array([n], "<u8").tobytes()
    try:
        with open(path, "wb") as f:
            f.write(hdr)
            f.write(rec.tobytes())
    except OSError as e:
        raise RuntimeError(f"{path}: cannot open for writing") from e


def _ck_header(path: str, raw: bytes):
    if len(raw) < 4 or raw[:4] != _CK_MAGIC:
        raise RuntimeError(f"{path}: bad checkpoint magic")
    if len(raw) < 8 or int(np.frombuffer(raw[4:8], "<u4")[0]) != _CK_VERSION:
        raise RuntimeError(f"{path}: unsupported checkpoint version")


def peek_checkpoint_hash(path: str) -> int:
    try:
        raw = open(path, "rb").read(16)
    except OSError as e:
        raise RuntimeError(f"{path}: cannot open") from e
    _ck_header(path, raw)
    if len(raw) < 16:
        raise RuntimeError(f"{path}: truncated checkpoint")
    return int(np.frombuffer(raw[8:16], "<u8")[0])


def load_checkpoint(path: str, expected_hash: int):
    """load_checkpoint: refuses on magic, version or config-hash mismatch."""
    from .optimizer import OptimState
    from .renderer import Scene
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise RuntimeError(f"{path}: cannot open") from e
    _ck_header(path, raw)
    if len(raw) < 40:
        raise RuntimeError(f"{path}: truncated checkpoint")
    if int(np.frombuffer(raw[8:16], "<u8")[0]) != (expected_hash & ((1 << 64) - 1)):
        raise RuntimeError(f"{path}: config hash mismatch: checkpoint was written with a different "
                           "effective configuration")
    it, nid = (int(x) for x in np.frombuffer(raw[16:32], "<i8"))
    n = int(np.frombuffer(raw[32:40], "<u8")[0])
    if len(raw) < 40 + n * _CK_REC.itemsize:
        raise RuntimeError(f"{path}: truncated checkpoint")
    rec = np.frombuffer(raw[40:40 + n * _CK_REC.itemsize], _CK_REC)
    sc = Scene(rec["center"].copy(), rec["rotation"].copy(), rec["radii"].copy(), rec["id"].copy())
    return OptimState(sc, rec["m"].copy(), rec["v"].copy(), rec["step"].copy(), rec["rgs"].copy(),
                      rec["rgc"].copy(), it, nid)
