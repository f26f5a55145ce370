"""CPU: pin the plain-C oracle (oracle/psplat_oracle.c) to the reference.

Two layers of pinning:
  * bit-for-bit agreement with the reference's own sources compiled through the
    Eigen shim (oracle/_ref) on the reference's fixture generators;
  * the reference's own known-answer tests, restated on the oracle:
    test_renderer.cpp, test_splatting.cpp, acceptance_main.cpp criteria 1-4.
"""
import numpy as np
import pytest

from oracle.oracle import Planes

LAMBDAS = [7.4, 40.0, 300.0]


def _same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def _fronto(z, r, cx=0.0, cy=0.0, n=1):
    P = Planes.empty(n)
    P.center[:] = [cx, cy, z]
    P.rotation[:] = [1, 0, 0, 0]
    P.radii[:] = r
    return P


def _stack(planes):
    return Planes(np.concatenate([p.center for p in planes]),
                  np.concatenate([p.rotation for p in planes]),
                  np.concatenate([p.radii for p in planes]),
                  np.arange(sum(p.n for p in planes), dtype=np.int64))


# ---------------------------------------------------------------- bit-exact vs reference
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("lam", LAMBDAS)
def test_restatement_bitwise_equal_to_reference(orc, ref, seed, lam):
    P = ref.random_scene(seed, 24)
    assert _same(P.center, orc.random_scene(seed, 24).center)
    cam = ref.make_view(32, 32, 24.0, True, seed)
    ocam = orc.make_view(32, 32, 24.0, True, seed)
    assert list(cam.rot_wc) == list(ocam.rot_wc) and list(cam.t_wc) == list(ocam.t_wc)
    td, tn = ref.fill_random_targets(cam, seed)
    otd, otn = orc.fill_random_targets(cam, seed)
    assert _same(td, otd) and _same(tn, otn)
    for a, b in zip(ref.bin_primitives(cam, P, lam), orc.bin_primitives(cam, P, lam)):
        assert _same(a, b)
    fr, lr, gr = ref.view_pass(cam, td, tn, P, lam)
    fo, lo, go = orc.view_pass(cam, td, tn, P, lam)
    for k in ("depth", "normal", "alpha", "rec_prim", "rec_count"):
        assert _same(fr[k], fo[k]), k
    assert lr["loss"] == lo["loss"]
    assert _same(lr["d_depth"], lo["d_depth"]) and _same(lr["d_normal"], lo["d_normal"])
    assert _same(gr, go)
    nr, no = ref.reference_render(cam, P, lam), orc.reference_render(cam, P, lam)
    for k in nr:
        assert _same(nr[k], no[k]), k


@pytest.mark.parametrize("seed", range(2000, 2020, 3))
def test_restatement_acceptance_scenes(orc, ref, seed):
    # acceptance_main.cpp:184-210: 8..64 planes, 32x32, lambda alternating 20/300
    from oracle.oracle import Oracle  # noqa: F401
    n = 8 + int(_splitmix_first(seed) % 57)
    lam = 20.0 if (seed - 2000) % 2 == 0 else 300.0
    P = ref.random_scene(seed, n)
    cam = ref.make_view(32, 32, 24.0, True, seed)
    fr = ref.render_view(cam, P, lam, keep_records=True)
    fo = orc.render_view(cam, P, lam, keep_records=True)
    for k in ("depth", "normal", "alpha", "rec_prim", "rec_count"):
        assert _same(fr[k], fo[k]), k


def _splitmix_first(seed):
    # TestRng(seed).next() of test_scenes.cpp:7-19
    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return x ^ (x >> 31)
    return sm(sm(seed))


def test_restatement_matches_reference_when_projection_overflows_int(orc, ref):
    # A plane straddling the camera's z=0 plane is clipped at z=1e-6 and projects
    # beyond 2^31 px; the reference's int() cast (renderer.cpp:108-111) then
    # yields an empty rect on x86-64. The restatement reproduces that.
    P = _stack([_fronto(2.0, 0.5), _fronto(0.0, 0.3, cx=0.5)])
    P.rotation[1] = [np.cos(0.7), np.sin(0.7), 0.0, 0.0]
    cam = ref.make_view(48, 32, 30.0)
    for lam in (7.4, 300.0):
        for a, b in zip(ref.bin_primitives(cam, P, lam), orc.bin_primitives(cam, P, lam)):
            assert _same(a, b)
        assert _same(ref.render_view(cam, P, lam)["depth"], orc.render_view(cam, P, lam)["depth"])


def test_restatement_big_view_c1(orc, ref):
    from paper_2412_03451_b200 import scenes
    wl = scenes.load("c1")
    from oracle.oracle import Camera, RefScenes
    c = wl.cams[0]
    cam = Camera()
    cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height = c.fx, c.fy, c.cx, c.cy, c.width, c.height
    for k in range(9):
        cam.rot_wc[k] = c.rot_wc[k]
    for k in range(3):
        cam.t_wc[k] = c.t_wc[k]
    td, tn = RefScenes().render_ground_truth(tuple(wl.room.tolist()[:3]) + (int(wl.room[3]), int(wl.room[4])),
                                             (Camera * 1)(cam))
    P = Planes(wl.scene.center, wl.scene.rotation, wl.scene.radii, wl.scene.ids)
    for lam in (7.3576, 300.0):
        fr, lr, gr = ref.view_pass(cam, td, tn, P, lam)
        fo, lo, go = orc.view_pass(cam, td, tn, P, lam)
        assert _same(fr["rec_prim"], fo["rec_prim"]) and _same(fr["depth"], fo["depth"])
        assert lr["loss"] == lo["loss"] and _same(gr, go)


# ---------------------------------------------------------------- test_renderer.cpp fixtures
def test_gather_single_plane_one_record(orc):  # test_renderer.cpp:35-47
    cam = orc.make_view(8, 8, 8.0)
    prim, z, w = orc.gather_intersections(cam, _fronto(2.0, 5.0), 300.0, 4, 4)
    assert len(prim) == 1 and abs(z[0] - 2.0) <= 2e-12 and w[0] == 1.0
    f = orc.render_view(cam, _fronto(2.0, 5.0), 300.0)
    assert np.allclose(f["normal"].reshape(-1, 3)[4 * 8 + 4], [0, 0, -1], atol=1e-12)


def test_gather_stacked_planes_depth_sorted(orc):  # test_renderer.cpp:49-59
    cam = orc.make_view(8, 8, 8.0)
    P = _stack([_fronto(3.0, 5.0), _fronto(2.0, 5.0)])
    prim, z, w = orc.gather_intersections(cam, P, 300.0, 3, 3)
    assert list(prim) == [1, 0] and abs(z[0] - 2.0) < 1e-12 and abs(z[1] - 3.0) < 1e-12


def test_gather_truncates_to_30_nearest(orc):  # test_renderer.cpp:61-73
    P = _stack([_fronto(1.0 + 0.05 * i, 5.0) for i in range(40)])
    cam = orc.make_view(4, 4, 4.0)
    prim, z, w = orc.gather_intersections(cam, P, 300.0, 1, 2)
    assert list(prim) == list(range(30)) and np.all(np.diff(z) >= 0)
    f = orc.render_view(cam, P, 300.0, keep_records=True)
    px = 2 * 4 + 1
    assert f["rec_count"][px] == 30 and list(f["rec_prim"][px * 30:(px + 1) * 30]) == list(range(30))


def test_fronto_plane_constant_depth(orc):  # test_renderer.cpp:98-108
    cam = orc.make_view(16, 12, 10.0)
    f = orc.render_view(cam, _fronto(2.0, 50.0), 300.0)
    assert np.allclose(f["depth"], 2.0, rtol=1e-12) and np.allclose(f["alpha"], 1.0, rtol=1e-12)


def test_zero_primitives_zero_maps(orc):  # test_renderer.cpp:110-117
    f = orc.render_view(orc.make_view(8, 8, 8.0), Planes.empty(0), 20.0)
    assert not f["depth"].any() and not f["alpha"].any()


def test_half_covering_plane_sharp_alpha(orc):  # test_renderer.cpp:119-135
    P = _fronto(2.0, 50.0, cx=-50.0)
    cam = orc.make_view(64, 16, 32.0)
    f = orc.render_view(cam, P, 300.0)
    for u in range(64):
        x_plane = (u + 0.5 - cam.cx) / cam.fx * 2.0
        a = f["alpha"][8 * 64 + u]
        if x_plane < -0.02:
            assert a >= 1 - 1e-4
        if x_plane > 0.02:
            assert a <= 1e-4


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_production_matches_naive(orc, seed):  # test_renderer.cpp:137-158
    P = orc.random_scene(seed, 24)
    cam = orc.make_view(32, 32, 24.0, True, seed)
    for lam in LAMBDAS:
        f, n = orc.render_view(cam, P, lam), orc.reference_render(cam, P, lam)
        assert max(np.abs(f[k] - n[k]).max() for k in n) < 1e-6


def _loss_setup(orc):
    cam = orc.make_view(1, 1, 1.0)
    td = np.array([3.0], np.float32)
    tn = np.array([0, 0, -1], np.float32)
    return cam, td, tn


@pytest.mark.parametrize("depth,normal,alpha,expect,dd", [
    (3.0, [0, 0, -1], 1.0, 0.0, 0.0),     # perfect fit
    (2.0, [0, 0, -1], 1.0, 1.0, -1.0),    # unit depth error costs alpha2
    (3.0, [0, 0, 1], 1.0, 20.0, 0.0),     # opposite normal costs alpha1 * 4
    (1.0, [0, 0, 1], 0.01, 0.0, 0.0),     # alpha below floor masks the pixel
])
def test_render_loss_fixtures(orc, depth, normal, alpha, expect, dd):  # test_renderer.cpp:160-203
    cam, td, tn = _loss_setup(orc)
    maps = {"depth": np.array([depth]), "normal": np.array(normal, float), "alpha": np.array([alpha])}
    lg = orc.render_loss(cam, td, tn, maps)
    assert abs(lg["loss"] - expect) <= 1e-12 * max(1.0, expect)
    assert lg["d_depth"][0] == dd


def _fd_check(orc, cfg, seed, n_prims, lam, rel=1e-3, abs_=1e-8, h=1e-5):
    P = orc.random_scene(seed, n_prims)
    cam = orc.make_view(8, 8, 8.0, True, seed)
    td, tn = orc.fill_random_targets(cam, seed)
    _, _, g = orc.view_pass(cam, td, tn, P, lam, cfg)
    bad = []
    for p in range(P.n):
        for k in range(11):
            fd = orc.fd_loss_gradient(cam, td, tn, P, p, k, lam, h, cfg)
            err = abs(g[p, k] - fd)
            r = err / max(abs(g[p, k]), abs(fd), 1e-300)
            if not (r < rel or err < abs_):
                bad.append((p, k, g[p, k], fd))
    return bad


@pytest.mark.parametrize("seed", [11, 12, 13, 14, 15])
def test_backward_matches_finite_differences(orc, seed):  # test_renderer.cpp:238-258
    cfg = orc.default_config()
    cfg.alpha_floor = 0.0
    assert _fd_check(orc, cfg, seed, 5, 10.0) == []


@pytest.mark.parametrize("seed", range(1000, 1050, 7))
def test_acceptance_criterion1_fd(orc, seed):  # acceptance_main.cpp:133-182 (subset)
    cfg = orc.default_config()
    cfg.alpha_floor = 0.0
    assert _fd_check(orc, cfg, seed, 5, 10.0) == []


def test_depth_only_center_gradient_sign(orc):  # test_renderer.cpp:260-285
    cfg = orc.default_config()
    cfg.alpha_floor, cfg.alpha1 = 0.0, 0.0
    cam = orc.make_view(8, 8, 8.0)
    td = np.full(64, 2.0, np.float32)
    tn = np.tile(np.array([0, 0, -1], np.float32), 64)
    P = _fronto(3.0, 4.0)
    _, _, g = orc.view_pass(cam, td, tn, P, 10.0, cfg)
    assert g[0, 2] > 0
    fd = orc.fd_loss_gradient(cam, td, tn, P, 0, 2, 10.0, 1e-5, cfg)
    assert abs(g[0, 2] - fd) < 1e-3 * abs(fd)


def test_out_of_frustum_and_occluded_get_zero_gradient(orc):  # test_renderer.cpp:287-326
    cam = orc.make_view(8, 8, 8.0)
    td, tn = orc.fill_random_targets(cam, 9)
    P = _stack([_fronto(2.0, 4.0), _fronto(-5.0, 1.0)])
    _, _, g = orc.view_pass(cam, td, tn, P, 20.0)
    assert not g[1].any()
    td, tn = orc.fill_random_targets(cam, 10)
    P = _stack([_fronto(2.0, 40.0), _fronto(3.0, 40.0)])
    f, _, g = orc.view_pass(cam, td, tn, P, 300.0)
    assert np.allclose(f["depth"], 2.0, rtol=1e-9) and not g[1].any()


def test_normalize_by_alpha_fd(orc):  # test_renderer.cpp:328-349
    cfg = orc.default_config()
    cfg.normalize_by_alpha = 1
    bad = _fd_check(orc, cfg, 21, 4, 10.0, abs_=1e-6)
    assert len(bad) <= 2


def test_nonfinite_gradient_raises_with_id(orc, ref):  # renderer.cpp:516-527
    P = _stack([_fronto(2.0, 1.0), _fronto(3.0, 1.0)])
    P.rotation[1] = 0.0  # q / |q| = NaN
    P.ids[:] = [70, 71]
    cam = orc.make_view(8, 8, 8.0)
    td, tn = orc.fill_random_targets(cam, 3)
    for o in (orc, ref):
        with pytest.raises(RuntimeError, match="primitive id 71"):
            o.view_pass(cam, td, tn, P, 20.0)


# ---------------------------------------------------------------- test_splatting.cpp fixtures
def test_splat_weight_fixtures(orc):  # test_splatting.cpp:39-62
    r = np.full(4, 0.5)
    ev = orc.plane_splat_weight(0.0, 0.0, r, 300.0)
    assert abs(ev["w_x"] - 2.0) <= 2e-12 and ev["weight"] == 1.0
    ev = orc.plane_splat_weight(0.5, 0.0, np.array([0.5, 0.5, 2.0, 2.0]), 300.0)
    assert ev["w_x"] == 1.0 and ev["weight"] == 1.0 and ev["x_selected"]
    ev = orc.plane_splat_weight(0.6, 0.0, r, 300.0)
    want = 2.0 / (1.0 + np.exp(150.0))  # doctest::Approx default: 100 float eps, relative
    assert ev["weight"] < 1e-4 and abs(ev["w_x"] - want) <= 1.2e-5 * max(abs(want), abs(ev["w_x"]))


def test_splat_weight_kernel_grid(orc):  # acceptance_main.cpp:212-266 (criterion 3)
    r = np.full(4, 0.5)
    xs = np.linspace(-0.7, 0.7, 201)
    g = np.array([[orc.plane_splat_weight(x, y, r, 300.0)["weight"] for x in xs] for y in xs])
    inner = (np.abs(xs)[None, :] <= 0.48) & (np.abs(xs)[:, None] <= 0.48)
    outer = (np.abs(xs)[None, :] >= 0.52) | (np.abs(xs)[:, None] >= 0.52)
    assert g[inner].min() >= 1 - 1e-4 and g[outer].max() <= 1e-4
    assert np.abs(g - g[:, ::-1]).max() <= 1e-12


def test_splat_partials_match_fd(orc):  # test_splatting.cpp:95-136
    rng = np.random.default_rng(202)
    checked = 0
    h = 1e-5
    for _ in range(500):
        r = rng.uniform(0.1, 0.8, 4)
        lam = rng.uniform(2.0, 40.0)
        px, py = rng.uniform(-1, 1, 2)
        ev = orc.plane_splat_weight(px, py, r, lam)
        raw = min(ev["w_x"], ev["w_y"])
        if abs(raw - 1) < 1e-3 or abs(ev["w_x"] - ev["w_y"]) < 1e-3 or min(abs(px), abs(py)) < 1e-3:
            continue
        k5 = 5 * lam
        if abs(k5 * (r[0 if px > 0 else 1] - abs(px))) > 20 or abs(k5 * (r[2 if py > 0 else 3] - abs(py))) > 20:
            continue
        checked += 1
        w = lambda qx, qy, rr: orc.plane_splat_weight(qx, qy, rr, lam)["weight"]  # noqa: E731
        fdx = (w(px + h, py, r) - w(px - h, py, r)) / (2 * h)
        assert abs(ev["d_px"] - fdx) < 1e-3 * max(abs(fdx), abs(ev["d_px"]), 1e-8)
        for k in range(4):
            up, dn = r.copy(), r.copy()
            up[k] += h
            dn[k] -= h
            fd = (w(px, py, up) - w(px, py, dn)) / (2 * h)
            assert abs(ev["d_radii"][k] - fd) < 1e-3 * max(abs(fd), abs(ev["d_radii"][k]), 1e-8)
    assert checked > 100


def test_lambda_schedule(orc, ref):  # test_splatting.cpp:176-189, acceptance crit. 4
    assert orc.lambda_schedule(0) == ref.lambda_schedule(0)
    assert abs(orc.lambda_schedule(0) - 7.357588823428847) < 1e-9
    assert abs(orc.lambda_schedule(1000) - 20.0) < 1e-9
    assert orc.lambda_schedule(3708) < 300.0 and orc.lambda_schedule(3709) == 300.0
    vals = [orc.lambda_schedule(i) for i in range(0, 5001)]
    assert all(b >= a for a, b in zip(vals, vals[1:]))
