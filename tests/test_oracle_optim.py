"""CPU: pin the optimiser restatement (oracle/psplat_oracle.c, "optimizer" part)
to the reference psplat::Optimizer (optimizer.cpp / optimizer.hpp) compiled
from its own sources, bit for bit, and restate the reference's known-answer
tests (test_optimizer.cpp) on it.
"""
import numpy as np
import pytest

from oracle.oracle import (OptimState, Planes, RefOptimizer, RestatedOptimizer,
                           default_optim_config)


def _same_state(a: OptimState, b: OptimState):
    for x, y in [(a.planes.center, b.planes.center), (a.planes.rotation, b.planes.rotation),
                 (a.planes.radii, b.planes.radii), (a.planes.ids, b.planes.ids), (a.m, b.m),
                 (a.v, b.v), (a.step, b.step), (a.rgs, b.rgs), (a.rgc, b.rgc)]:
        assert x.shape == y.shape and np.array_equal(x, y)
    assert a.iteration == b.iteration and a.next_id == b.next_id


def _setup(o, seed=5, n=6, n_views=1, size=16):
    P = o.random_scene(seed, n)
    cams, tg = [], []
    for k in range(n_views):
        cam = o.make_view(size, size, 12.0, True, seed + k)
        cams.append(cam)
        tg.append(o.fill_random_targets(cam, seed + k))
    return P, cams, tg


def test_default_optim_config_matches(ref, orc):
    a, b = default_optim_config(ref), default_optim_config(orc)
    for f, _ in a._fields_:
        assert getattr(a, f) == getattr(b, f), f


@pytest.mark.parametrize("seed", [0, 7, 123456789])
def test_view_for_slot_matches_reference(ref, orc, seed):
    P, cams, tg = _setup(orc, n_views=1)
    for n_views in (1, 5, 32):
        cams_n = [cams[0]] * n_views
        tg_n = [tg[0]] * n_views
        oc = default_optim_config(orc)
        oc.seed = seed
        r = RefOptimizer(ref, P, cams_n, tg_n, oc)
        s = RestatedOptimizer(orc, OptimState.fresh(P), cams_n, tg_n, oc)
        got = [s.view_for_slot(k) for k in range(4 * n_views + 3)]
        want = [r.view_for_slot(k) for k in range(4 * n_views + 3)]
        assert got == want
        # every epoch is a permutation
        for e in range(4):
            assert sorted(got[e * n_views:(e + 1) * n_views]) == list(range(n_views))


@pytest.mark.parametrize("views_per_step,single_radii", [(1, False), (3, False), (2, True)])
def test_adam_steps_bitwise_vs_reference(ref, orc, views_per_step, single_radii):
    P, cams, tg = _setup(orc, seed=5, n=6, n_views=4)
    oc = default_optim_config(orc)
    oc.enable_split = 0
    oc.lr_radii = 0.05  # test_optimizer.cpp:96: push radii toward the floor
    oc.views_per_step = views_per_step
    oc.single_radii = int(single_radii)
    oc.seed = 3
    r = RefOptimizer(ref, P, cams, tg, oc)
    s = RestatedOptimizer(orc, OptimState.fresh(P), cams, tg, oc)
    for it in range(12):
        lr, ls = r.step(), s.step()
        assert lr == ls, it
        assert np.array_equal(r.last_grads(), s.last_grads)
        _same_state(r.state(), s.st)


def test_maybe_split_bitwise_vs_reference(ref, orc):
    P, cams, tg = _setup(orc, seed=11, n=40, n_views=1)
    rng = np.random.default_rng(4)
    oc = default_optim_config(orc)
    for it in (999, 1000, 2000):
        r = RefOptimizer(ref, P, cams, tg, oc)
        s = RestatedOptimizer(orc, OptimState.fresh(P), cams, tg, oc)
        rgs = rng.uniform(0.0, 0.6, (P.n, 4))
        rgc = rng.integers(0, 3, P.n).astype(np.int64)
        rgs[rgc == 0] = 0.0
        rgs[5] = [0.3, 0.3, 0.3, 0.3]  # mean_x == mean_y: X wins (optimizer.cpp:158)
        rgc[5] = 1
        r.set_stats(it, rgs, rgc)
        s.st.iteration, s.st.rgs, s.st.rgc = it, rgs.copy(), rgc.copy()
        kr, ks = r.maybe_split(), s.maybe_split()
        assert kr == ks and (it != 1000 or kr > 0)
        st = r.state()
        if it % 1000 != 0:  # not fired: statistics untouched
            assert np.array_equal(st.rgs, rgs) and np.array_equal(st.rgc, rgc)
            continue
        _same_state(st, s.st)
        # then Adam keeps agreeing on the grown scene
        assert r.step() == s.step()
        _same_state(r.state(), s.st)


# ---- test_optimizer.cpp restated on the restatement
def test_zero_gradients_leave_parameters_unchanged(orc):  # test_optimizer.cpp:59-74
    P = Planes.empty(1)
    P.center[0] = [0, 0, 2]
    P.rotation[0] = [1, 0, 0, 0]
    P.radii[0] = 0.5
    cam = orc.make_view(8, 8, 8.0)
    tg = (np.zeros(64, np.float32), np.zeros(192, np.float32))
    oc = default_optim_config(orc)
    oc.enable_split = 0
    s = RestatedOptimizer(orc, OptimState.fresh(P), [cam], [tg], oc)
    assert s.step() == 0.0
    assert np.array_equal(s.st.planes.center, P.center)
    assert np.array_equal(s.st.planes.rotation, P.rotation)
    assert np.array_equal(s.st.planes.radii, P.radii)
    assert not s.st.m.any()


def test_plane_behind_target_moves_toward_camera(orc):  # test_optimizer.cpp:76-90
    P = Planes.empty(1)
    P.center[0] = [0, 0, 3]
    P.rotation[0] = [1, 0, 0, 0]
    P.radii[0] = 4.0
    cam = orc.make_view(8, 8, 8.0)
    tn = np.zeros(192, np.float32)
    tn[2::3] = -1.0
    oc = default_optim_config(orc)
    oc.enable_split = 0
    s = RestatedOptimizer(orc, OptimState.fresh(P), [cam], [(np.full(64, 2.0, np.float32), tn)], oc)
    s.step()
    assert s.st.planes.center[0, 2] < 3.0


def test_quaternions_unit_radii_floor(orc):  # test_optimizer.cpp:92-104
    P, cams, tg = _setup(orc, seed=5, n=6)
    oc = default_optim_config(orc)
    oc.enable_split = 0
    oc.lr_radii = 0.05
    s = RestatedOptimizer(orc, OptimState.fresh(P), cams, tg, oc)
    for _ in range(25):
        s.step()
    assert np.all(np.abs(np.linalg.norm(s.st.planes.rotation, axis=1) - 1.0) < 1e-6)
    assert np.all(s.st.planes.radii >= 1e-4)


def test_split_x_gradient_tiles_exactly(orc):  # test_optimizer.cpp:120-157
    P = Planes.empty(1)
    P.center[0] = [0, 0, 0]
    P.rotation[0] = [1, 0, 0, 0]
    P.radii[0] = [1.0, 1.0, 0.5, 0.5]
    cam = orc.make_view(4, 4, 4.0)
    tg = (np.zeros(16, np.float32), np.zeros(48, np.float32))
    oc = default_optim_config(orc)
    oc.split_interval = 10
    s = RestatedOptimizer(orc, OptimState.fresh(P), [cam], [tg], oc)
    s.st.iteration = 10
    s.st.rgs[0] = [0.5, 0.5, 0.0, 0.0]
    s.st.rgc[0] = 1
    assert s.maybe_split() == 1
    c, r = s.st.planes.center, s.st.planes.radii
    assert s.st.planes.n == 2 and list(s.st.planes.ids) == [1, 2]
    assert np.allclose(c[0], [0.5, 0, 0]) and np.allclose(c[1], [-0.5, 0, 0])
    assert np.allclose(r, [[0.5, 0.5, 0.5, 0.5]] * 2)
    assert not s.st.rgs.any() and not s.st.rgc.any()


# ---- merge_planes (optimizer.cpp:236-299), rect_distance (geometry.cpp:131-149)
def _make_prim(P, i, center, q, radii, pid):
    q = np.asarray(q, np.float64)
    P.center[i] = center
    P.rotation[i] = q / np.sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]))
    P.radii[i] = radii
    P.ids[i] = pid


def _two_rect_scene(hinge_deg):  # test_optimizer.cpp:207-220
    P = Planes.empty(2)
    _make_prim(P, 0, [0, 0, 0], [1, 0, 0, 0], [0.5] * 4, 0)
    th = hinge_deg * np.pi / 180.0
    _make_prim(P, 1, [0.5 + 0.5 * np.cos(th), 0.0, 0.5 * np.sin(th)],
               [np.cos(-th / 2), 0, np.sin(-th / 2), 0], [0.5] * 4, 1)
    return P


def test_merge_reference_cases(orc):  # test_optimizer.cpp:224-261
    m = orc.merge_planes(_two_rect_scene(0.0), (0.5, 0, 0))
    assert m["n"] == 1 and abs(abs(m["normal"][0, 2]) - 1.0) < 1e-12
    assert orc.merge_planes(_two_rect_scene(24.9), (0.5, 0, 0))["n"] == 1
    assert orc.merge_planes(_two_rect_scene(25.1), (0.5, 0, 0))["n"] == 2
    P = Planes.empty(2)
    _make_prim(P, 0, [0, 0, 0], [1, 0, 0, 0], [0.5] * 4, 0)
    _make_prim(P, 1, [0, 0, 0.5], [1, 0, 0, 0], [0.5] * 4, 1)
    assert orc.merge_planes(P, use_adjacency=False)["n"] == 2
    P.center[1, 2] = 0.09
    assert orc.merge_planes(P, use_adjacency=False)["n"] == 1
    P.center[1, 2] = 0.11
    assert orc.merge_planes(P, use_adjacency=False)["n"] == 2
    P.center[1] = [3, 0, 0]
    assert orc.merge_planes(P)["n"] == 2
    assert orc.merge_planes(P, use_adjacency=False)["n"] == 1


def _same_merge(a, b):
    assert a["n"] == b["n"]
    for k in ("instance_of", "normal", "offset", "area"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("seed", [1, 88, 4242])
def test_merge_bitwise_vs_reference_random(ref, orc, seed):
    rng = np.random.default_rng(seed)
    n = 120
    P = Planes.empty(n)
    for i in range(n):
        q = rng.normal(size=4)
        _make_prim(P, i, rng.uniform(-2, 2, 3), q, rng.uniform(0.1, 0.6, 4), 1000 - i)
    for use_adj in (True, False):
        for gate in (25.0, 60.0):
            a = ref.merge_planes(P, (0.1, -0.2, 0.3), gate, 0.3, 0.2, use_adj)
            b = orc.merge_planes(P, (0.1, -0.2, 0.3), gate, 0.3, 0.2, use_adj)
            _same_merge(a, b)
    # rect_distance on its own, including touching / crossing / parallel pairs
    for i in range(0, n - 1, 3):
        a = [P.center[i], P.rotation[i], P.radii[i], P.center[i + 1], P.rotation[i + 1], P.radii[i + 1]]
        assert ref.rect_distance(*a) == orc.rect_distance(*a)


def test_merge_bitwise_vs_reference_room(ref, orc):
    """Depth-initialised planes of the C2 room: walls tiled by many near-coplanar planes."""
    from paper_2412_03451_b200 import scenes
    wl = scenes.load("c2")
    s = wl.scene
    P = Planes(s.center.copy(), s.rotation.copy(), s.radii.copy(), s.ids.copy())
    sc = P.center.mean(axis=0)
    a = ref.merge_planes(P, sc)
    b = orc.merge_planes(P, sc)
    _same_merge(a, b)
    assert 1 < a["n"] < P.n
