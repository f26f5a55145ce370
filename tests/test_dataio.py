"""CPU: the PSMP dataset loader (psg_dataset_*, psg_*_map_f32) against the format
of dataio.hpp:12-14 / dataio.cpp:19-254, restating test_dataio.cpp, and against the
reference's own dataio.cpp: it is compiled into oracle/_ref through test-only
nlohmann/json and libpng header shims (oracle/json_shim, oracle/png_shim), so the
reference writes datasets and maps that the repo's loader must read bit for bit,
the repo's writer must produce byte-identical files, and each side reads the
other's output.
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


# ---------------------------------------------------------------- vs the reference's dataio.cpp
def _refio():
    from oracle.oracle import LIBS, RefDataIO
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefDataIO()


def _room_views(n=6):
    """Views of the reference's own synthetic room (generate_box_room(4,4,3,1,13),
    sample_trajectory, render_ground_truth: tests/test_dataio.cpp:30-45), 16x12."""
    from oracle.oracle import LIBS, RefScenes
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from oracle.oracle import Camera
    rs = RefScenes()
    allc = rs.room_views(4, 4, 3, 1, 13, 35, 13, 16, 12)  # coverage needs 35 poses; first n kept
    cams = (Camera * n)(*[allc[i] for i in range(n)])
    td, tn = rs.render_ground_truth((4, 4, 3, 1, 13), cams)
    faces = rs.room_faces(4, 4, 3, 1, 13)
    return [cams[i] for i in range(n)], td, tn, faces


def _as_views(cams, td, tn):
    out, o = [], 0
    for i, c in enumerate(cams):
        m = c.width * c.height
        out.append(CameraView(c.fx, c.fy, c.cx, c.cy, c.width, c.height,
                              np.array(list(c.rot_wc)).reshape(3, 3), np.array(list(c.t_wc)),
                              td[o:o + m].copy(), tn[3 * o:3 * (o + m)].copy(), id=i))
        o += m
    return out


def _faces_meta(faces):
    return [GtFace(int(f[14]), f[0:3].copy(), f[3:6].copy(), f[6:9].copy(), float(f[9]), float(f[10]))
            for f in faces]


def _tree_bytes(root):
    out = {}
    for d, _, files in os.walk(root):
        for f in files:
            p = os.path.join(d, f)
            out[os.path.relpath(p, root)] = open(p, "rb").read()
    return out


def test_reference_written_dataset_loads_bitwise(tmp_path):
    """load_dataset (dataio.cpp:136-201) of a dataset the reference's write_dataset
    produced: cameras, ids, targets and meta identical to what the reference's own
    load_dataset returns, with and without stride."""
    io = _refio()
    cams, td, tn, faces = _room_views(6)
    root = str(tmp_path / "ref")
    io.write_dataset(root, cams, np.arange(6) * 3 + 1, td, tn, (2.0, 2.0, 1.5), "meters", faces)
    for stride in (1, 2, 4):
        want = io.load_dataset(root, stride)
        ds = Dataset(root, stride)
        assert ds.n_views == len(want["cams"])
        got_td, got_tn = ds.read()
        assert np.array_equal(got_td, want["td"]) and np.array_equal(got_tn, want["tn"])
        assert np.array_equal(ds.ids, want["ids"])
        for a, b in zip(ds.cameras(), want["cams"]):
            assert (a.fx, a.fy, a.cx, a.cy, a.width, a.height) == (b.fx, b.fy, b.cx, b.cy, b.width, b.height)
            assert list(a.rot_wc) == list(b.rot_wc) and list(a.t_wc) == list(b.t_wc)
        assert ds.has_meta and want["has_meta"]
        assert np.array_equal(ds.meta.scene_center, want["scene_center"]) and ds.meta.units == want["units"]
        assert len(ds.meta.gt_faces) == len(want["faces"]) == len(faces)
        for f, w in zip(ds.meta.gt_faces, want["faces"]):
            assert f.instance_id == int(w[14]) and f.half_u == w[9] and f.half_v == w[10]
            assert np.array_equal(f.center, w[0:3]) and np.array_equal(f.u_axis, w[3:6])
            assert np.array_equal(f.v_axis, w[6:9]) and np.array_equal(f.normal, w[11:14])
        ds.close()


def test_writers_byte_identical_and_cross_readable(tmp_path):
    """write_dataset (dataio.cpp:203-254): the repo's writer and the reference's
    writer produce byte-identical trees (cameras.txt at 17 digits, PSMP maps,
    meta.json as nlohmann dump(2) with sorted keys) for the same views, and the
    reference's load_dataset reads the repo-written dataset back bit for bit."""
    io = _refio()
    cams, td, tn, faces = _room_views(5)
    views = _as_views(cams, td, tn)
    a, b = str(tmp_path / "repo"), str(tmp_path / "ref")
    write_dataset(a, views, SceneMeta(np.array([2.0, 2.0, 1.5]), "meters", _faces_meta(faces)))
    io.write_dataset(b, cams, np.arange(5), td, tn, (2.0, 2.0, 1.5), "meters", faces)
    ta, tb = _tree_bytes(a), _tree_bytes(b)
    assert sorted(ta) == sorted(tb)
    for k in ta:
        assert ta[k] == tb[k], k
    back = io.load_dataset(a)
    assert np.array_equal(back["td"], td) and np.array_equal(back["tn"], tn)


def test_maps_cross_read_and_reference_errors(tmp_path):
    """write_map_f32 / read_map_f32 (dataio.cpp:65-97): byte-identical files from
    both writers; each reader reads the other's; the reference rejects what the repo
    rejects (truncated payload, wrong magic, wrong channel count), path in message."""
    io = _refio()
    data = np.array([0.5, -1.25, 3.75, 1e-20, 1e20, 0.0], np.float32)
    pa, pb = str(tmp_path / "a.f32"), str(tmp_path / "b.f32")
    write_map_f32(pa, 3, 2, 1, data)
    io.write_map_f32(pb, 3, 2, 1, data)
    assert open(pa, "rb").read() == open(pb, "rb").read()
    w, h, got = io.read_map_f32(pa, 1)
    assert (w, h) == (3, 2) and np.array_equal(got, data)
    w, h, got = read_map_f32(pb, 1)
    assert (w, h) == (3, 2) and np.array_equal(got, data)
    raw = open(pa, "rb").read()
    bad = {"trunc.f32": raw[:-5], "magic.f32": b"NOPE" + bytes(12)}
    for name, blob in bad.items():
        p = str(tmp_path / name)
        open(p, "wb").write(blob)
        with pytest.raises(RuntimeError, match=name):
            io.read_map_f32(p, 1)
        with pytest.raises(RuntimeError, match=name):
            read_map_f32(p, 1)
    for reader in (io.read_map_f32, read_map_f32):
        with pytest.raises(RuntimeError, match="a.f32"):
            reader(pa, 3)


def test_reference_and_repo_reject_the_same_datasets(tmp_path):
    """validate_view and the loader's checks (dataio.cpp:120-201) on broken datasets
    the reference itself wrote: both loaders refuse each one."""
    io = _refio()
    cams, td, tn, faces = _room_views(3)
    base = str(tmp_path / "base")
    io.write_dataset(base, cams, np.arange(3), td, tn, (0.0, 0.0, 0.0), "meters", faces)
    import shutil

    def variant(name, fn):
        d = str(tmp_path / name)
        shutil.copytree(base, d)
        fn(d)
        return d

    cases = [
        variant("missing_normal", lambda d: os.remove(os.path.join(d, "normal", "1.f32"))),
        variant("bad_line", lambda d: open(os.path.join(d, "cameras.txt"), "w").write("0 bad line\n")),
        variant("empty", lambda d: open(os.path.join(d, "cameras.txt"), "w").write("# no cameras\n")),
        variant("bad_meta", lambda d: open(os.path.join(d, "meta.json"), "w").write("{not json")),
    ]

    def nonunit(d):
        p = os.path.join(d, "normal", "0.f32")
        w, h, n = io.read_map_f32(p, 3)
        n[n != 0] *= 1.01
        io.write_map_f32(p, w, h, 3, n)
    cases.append(variant("nonunit_normal", nonunit))

    def wrong_res(d):
        p = os.path.join(d, "depth", "2.f32")
        io.write_map_f32(p, 8, 6, 1, np.ones(48, np.float32))
    cases.append(variant("wrong_res", wrong_res))
    for d in cases:
        with pytest.raises(RuntimeError):
            io.load_dataset(d)
        with pytest.raises(RuntimeError):
            ds = Dataset(d)
            ds.read()
    with pytest.raises(ValueError):
        io.load_dataset(base, 0)
    with pytest.raises(ValueError):
        Dataset(base, 0)
