"""CPU: the PSMP dataset loader (psg_dataset_*, psg_*_map_f32) against the format
of dataio.hpp:12-14 / dataio.cpp:19-248, restating test_dataio.cpp.

The reference's dataio.cpp needs nlohmann/json and libpng, which are absent, so it
cannot be built as an oracle here; the contract is the documented byte format
(checked against raw bytes below) and the reference's own tests and messages.
"""
import os
import struct

import numpy as np
import pytest

from paper_2412_03451_b200 import CameraView, Dataset, SceneMeta, read_map_f32, write_dataset, write_map_f32
from paper_2412_03451_b200.dataio import GtFace


def _views(n, w=16, h=12, seed=3):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        a, b, c, d = q
        R = np.array([[1 - 2 * (c * c + d * d), 2 * (b * c - a * d), 2 * (b * d + a * c)],
                      [2 * (b * c + a * d), 1 - 2 * (b * b + d * d), 2 * (c * d - a * b)],
                      [2 * (b * d - a * c), 2 * (c * d + a * b), 1 - 2 * (b * b + c * c)]])
        td = rng.uniform(0.5, 4.0, w * h).astype(np.float32)
        td[::7] = 0.0
        nn = rng.normal(size=(w * h, 3))
        nn /= np.linalg.norm(nn, axis=1, keepdims=True)
        tn = nn.astype(np.float32).reshape(-1)
        tn[3 * 5:3 * 6] = 0.0
        out.append(CameraView(10.0 + i / 3, 10.0, w / 2 + 0.1, h / 2, w, h, R,
                              rng.normal(size=3), td, tn, id=i))
    return out


def test_map_round_trip_bitwise_and_bytes(tmp_path):  # test_dataio.cpp:56-69
    data = np.array([0.5, -1.25, 3.75, 1e-20, 1e20, 0.0], np.float32)
    p = str(tmp_path / "m.f32")
    write_map_f32(p, 3, 2, 1, data)
    raw = open(p, "rb").read()
    assert raw[:4] == b"PSMP" and struct.unpack("<III", raw[4:16]) == (1, 3, 2)
    assert raw[16:] == data.tobytes()
    w, h, got = read_map_f32(p, 1)
    assert (w, h) == (3, 2) and got.tobytes() == data.tobytes()


def test_map_truncated_wrong_magic_wrong_channels(tmp_path):  # test_dataio.cpp:71-97
    p = str(tmp_path / "trunc.f32")
    write_map_f32(p, 4, 3, 1, np.ones(12, np.float32))
    os.truncate(p, os.path.getsize(p) - 5)
    with pytest.raises(RuntimeError, match="trunc.f32"):
        read_map_f32(p, 1)
    bad = tmp_path / "bad.f32"
    bad.write_bytes(b"NOPE" + b"\0" * 12)
    with pytest.raises(RuntimeError, match="bad map magic"):
        read_map_f32(str(bad), 1)
    one = str(tmp_path / "one.f32")
    write_map_f32(one, 3, 2, 1, np.zeros(6, np.float32))
    with pytest.raises(RuntimeError, match="payload length does not match header"):
        read_map_f32(one, 3)
    ver = tmp_path / "ver.f32"
    ver.write_bytes(b"PSMP" + struct.pack("<III", 2, 1, 1) + b"\0" * 4)
    with pytest.raises(RuntimeError, match="unsupported map version"):
        read_map_f32(str(ver), 1)


def test_dataset_round_trip_bitwise(tmp_path):  # test_dataio.cpp:99-118
    views = _views(4)
    write_dataset(str(tmp_path), views, SceneMeta(np.array([2.0, 2.0, 1.5])))
    ds = Dataset(str(tmp_path))
    got = ds.views(threads=3)
    assert len(got) == 4 and list(ds.ids) == [0, 1, 2, 3]
    for a, b in zip(views, got):
        assert a.target_depth.tobytes() == b.target_depth.tobytes()
        assert a.target_normal.tobytes() == b.target_normal.tobytes()
        assert (a.fx, a.fy, a.cx, a.cy, a.width, a.height) == (b.fx, b.fy, b.cx, b.cy, b.width, b.height)
        assert np.array_equal(np.asarray(a.rot_wc), b.rot_wc) and np.array_equal(a.t_wc, b.t_wc)
    assert ds.has_meta and np.array_equal(ds.meta.scene_center, [2.0, 2.0, 1.5])
    # threads do not change the bytes
    assert all(x.tobytes() == y.tobytes() for x, y in zip(ds.read(threads=1), ds.read(threads=8)))


def test_dataset_stride(tmp_path):  # test_dataio.cpp:120-127
    write_dataset(str(tmp_path), _views(8), SceneMeta())
    assert Dataset(str(tmp_path), 2).n_views == 4
    assert list(Dataset(str(tmp_path), 2).ids) == [0, 2, 4, 6]
    assert Dataset(str(tmp_path), 8).n_views == 1
    with pytest.raises(ValueError):
        Dataset(str(tmp_path), 0)


def test_dataset_missing_files_and_malformed_lines(tmp_path):  # test_dataio.cpp:129-139
    write_dataset(str(tmp_path), _views(2), SceneMeta())
    os.remove(tmp_path / "normal" / "1.f32")
    with pytest.raises(RuntimeError, match="1.f32"):
        Dataset(str(tmp_path))
    (tmp_path / "cameras.txt").write_text("0 bad line\n")
    with pytest.raises(RuntimeError, match="malformed camera line"):
        Dataset(str(tmp_path))
    (tmp_path / "cameras.txt").write_text("# only a comment\n")
    with pytest.raises(RuntimeError, match="no cameras loaded"):
        Dataset(str(tmp_path))
    with pytest.raises(RuntimeError, match="cannot open"):
        Dataset(str(tmp_path / "nowhere"))


def test_dataset_validation(tmp_path):  # validate_view, dataio.cpp:107-121
    v = _views(1)
    v[0].rot_wc = np.asarray(v[0].rot_wc) * 1.01
    write_dataset(str(tmp_path / "a"), v, SceneMeta())
    with pytest.raises(RuntimeError, match="pose rotation not orthonormal"):
        Dataset(str(tmp_path / "a")).read()
    v = _views(1)
    v[0].target_normal = v[0].target_normal.copy()
    v[0].target_normal[3 * 9:3 * 10] *= 1.01
    write_dataset(str(tmp_path / "b"), v, SceneMeta())
    with pytest.raises(RuntimeError, match="non-unit target normal"):
        Dataset(str(tmp_path / "b")).read()
    v = _views(1)
    write_dataset(str(tmp_path / "c"), v, SceneMeta())
    write_map_f32(str(tmp_path / "c" / "depth" / "0.f32"), 12, 16, 1, v[0].target_depth)
    with pytest.raises(RuntimeError, match="resolution differs from cameras.txt"):
        Dataset(str(tmp_path / "c"))


def test_dataset_gt_faces_meta(tmp_path):  # test_dataio.cpp:141-164
    faces = [GtFace(3, np.array([1.0, 2.0, 3.0]), np.array([1.0, 0, 0]), np.array([0, 1.0, 0]), 0.5, 0.25)]
    write_dataset(str(tmp_path), _views(1), SceneMeta(np.zeros(3), "meters", faces))
    ds = Dataset(str(tmp_path))
    f = ds.meta.gt_faces[0]
    assert f.instance_id == 3 and f.half_u == 0.5 and f.half_v == 0.25
    assert np.array_equal(f.normal, [0, 0, 1.0])


def test_checkpoint_round_trip_and_refusals(tmp_path):  # dataio.cpp:250-330
    from paper_2412_03451_b200 import OptimState, Scene, load_checkpoint, peek_checkpoint_hash, save_checkpoint
    rng = np.random.default_rng(5)
    n = 7
    st = OptimState(Scene(rng.normal(size=(n, 3)), rng.normal(size=(n, 4)), rng.uniform(0.1, 1, (n, 4)),
                          np.arange(10, 10 + n)),
                    rng.normal(size=(n, 11)), rng.uniform(size=(n, 11)), rng.integers(0, 99, n),
                    rng.uniform(size=(n, 4)), rng.integers(0, 9, n), 1234, 17)
    p = str(tmp_path / "s.psck")
    save_checkpoint(p, st, 0xDEADBEEFCAFEF00D)
    raw = open(p, "rb").read()
    assert raw[:4] == b"PSCK" and len(raw) == 40 + n * (8 * (1 + 3 + 4 + 4 + 1 + 11 + 11 + 4 + 1))
    assert peek_checkpoint_hash(p) == 0xDEADBEEFCAFEF00D
    got = load_checkpoint(p, 0xDEADBEEFCAFEF00D)
    assert got.iteration == 1234 and got.next_id == 17
    for a, b in [(got.scene.center, st.scene.center), (got.scene.ids, st.scene.ids), (got.m, st.m),
                 (got.v, st.v), (got.step, st.step), (got.radii_grad_sum, st.radii_grad_sum),
                 (got.radii_grad_count, st.radii_grad_count), (got.scene.radii, st.scene.radii)]:
        assert np.array_equal(a, b)
    with pytest.raises(RuntimeError, match="config hash mismatch"):
        load_checkpoint(p, 1)
    os.truncate(p, len(raw) - 3)
    with pytest.raises(RuntimeError, match="truncated checkpoint"):
        load_checkpoint(p, 0xDEADBEEFCAFEF00D)
    (tmp_path / "bad").write_bytes(b"XXXX" + b"\0" * 40)
    with pytest.raises(RuntimeError, match="bad checkpoint magic"):
        load_checkpoint(str(tmp_path / "bad"), 0)
