"""GPU: the device optimiser (psg_optim_*) against the
optimiser restatement (oracle/psplat_oracle.c, pinned bitwise to the reference
psplat::Optimizer by tests/test_oracle_optim.py) and the reference itself.

Contract:
  * Adam + renormalisation + clamp + radii sums (optimizer.cpp:84-140) given the
    same gradients: bit-identical, including steps where the host libm's pow
    is not correctly rounded (the bias table comes from the host libm);
  * maybe_split (optimizer.cpp:142-202): bit-identical scene, ids, Adam state;
  * the full device Optimizer::step (fp64 renderer) vs the reference Optimizer:
    loss within 1e-12 relative and parameters within 1e-9 relative per step
    (the only difference is the gradient summation order, ~1e-16).
"""
import ctypes as C

import numpy as np
import pytest

from _util import to_scene, to_view
from oracle.oracle import OptimState, Planes, RefOptimizer, RestatedOptimizer, default_optim_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    return True


def _views(orc, cams, tg):
    from paper_2412_03451_b200 import CameraView
    out = []
    for cam, (td, tn) in zip(cams, tg):
        v = to_view(cam)
        out.append(CameraView(v.fx, v.fy, v.cx, v.cy, v.width, v.height, v.rot_wc, v.t_wc, td, tn))
    return out


def _setup(orc, seed=5, n=6, n_views=4, size=16):
    P = orc.random_scene(seed, n)
    cams, tg = [], []
    for k in range(n_views):
        cam = orc.make_view(size, size, 12.0, True, seed + k)
        cams.append(cam)
        tg.append(orc.fill_random_targets(cam, seed + k))
    return P, cams, tg


def _ocfg(oc_orc, **kw):
    from paper_2412_03451_b200 import OptimConfig
    o = OptimConfig()
    for f in ("lr_center", "lr_radii", "lr_rotation", "beta1", "beta2", "eps", "split_interval",
              "split_grad_threshold", "views_per_step", "seed", "radii_floor"):
        setattr(o, f, getattr(oc_orc, f))
    o.enable_split = bool(oc_orc.enable_split)
    o.single_radii = bool(oc_orc.single_radii)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _dev_state_equal(dev, st: OptimState, exact=True, rtol=0.0):
    s = dev.state()
    pairs = [(s.scene.center, st.planes.center), (s.scene.rotation, st.planes.rotation),
             (s.scene.radii, st.planes.radii), (s.m, st.m), (s.v, st.v),
             (s.radii_grad_sum, st.rgs)]
    for a, b in pairs:
        assert a.shape == b.shape
        if exact:
            assert np.array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=rtol, atol=rtol * max(np.abs(b).max(), 1e-300))
    assert np.array_equal(s.scene.ids, st.planes.ids)
    assert np.array_equal(s.step, st.step) and np.array_equal(s.radii_grad_count, st.rgc)
    assert s.iteration == st.iteration and s.next_id == st.next_id


@pytest.mark.parametrize("single_radii", [False, True])
def test_adam_apply_bitwise(gpu, orc, single_radii):
    from paper_2412_03451_b200 import Optimizer
    P, cams, tg = _setup(orc, n=300, n_views=1)
    oc = default_optim_config(orc)
    oc.single_radii = int(single_radii)
    oc.lr_radii = 0.05
    dev = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    st = OptimState.fresh(P)
    L = orc.lib
    rng = np.random.default_rng(1)
    # resume at Adam step 2900 so the updates cross s = 2904, a step where
    # glibc's pow(0.999, s) is not the correctly rounded value
    st.step[:] = 2900
    st.m[:] = rng.normal(0, 1e-3, st.m.shape)
    st.v[:] = rng.uniform(0, 1e-5, st.v.shape)
    from paper_2412_03451_b200 import OptimState as DevState
    dev.load_state(DevState(to_scene(P), st.m, st.v, st.step, st.rgs, st.rgc, 0, st.next_id))
    d = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    i64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    for it in range(8):
        g = rng.normal(0, 10.0 ** rng.integers(-6, 1), (P.n, 11))
        g[::7] = 0.0
        dev.set_gradients(g)
        dev.apply()
        L.orc_accumulate_radii_grads(C.c_int64(P.n), d(g), d(st.rgs), i64(st.rgc))
        Pp = st.planes
        L.orc_apply_adam(C.c_int64(P.n), d(Pp.center), d(Pp.rotation), d(Pp.radii), d(st.m),
                         d(st.v), i64(st.step), d(g), C.byref(oc))
        _dev_state_equal(dev, st)


def test_maybe_split_bitwise(gpu, orc):
    from paper_2412_03451_b200 import Optimizer
    from paper_2412_03451_b200 import OptimState as DevState
    P, cams, tg = _setup(orc, seed=11, n=500, n_views=2)
    oc = default_optim_config(orc)
    rng = np.random.default_rng(4)
    for it in (999, 1000):
        dev = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
        s = RestatedOptimizer(orc, OptimState.fresh(P), cams, tg, oc)
        rgs = rng.uniform(0.0, 0.6, (P.n, 4))
        rgc = rng.integers(0, 3, P.n).astype(np.int64)
        rgs[rgc == 0] = 0.0
        s.st.iteration, s.st.rgs, s.st.rgc = it, rgs.copy(), rgc.copy()
        s.st.m[:] = rng.normal(0, 1e-3, s.st.m.shape)
        s.st.step[:] = 7
        dev.load_state(DevState(to_scene(P), s.st.m, s.st.v, s.st.step, rgs, rgc, it, s.st.next_id))
        k_dev, k_orc = dev.maybe_split(), s.maybe_split()
        assert k_dev == k_orc and (it != 1000 or k_dev > 0)
        if it == 1000:
            assert dev.n_planes == P.n + k_dev
            _dev_state_equal(dev, s.st)
        else:
            sd = dev.state()
            assert np.array_equal(sd.radii_grad_sum, rgs) and sd.scene.n == P.n


@pytest.mark.parametrize("views_per_step", [1, 3])
def test_optimizer_steps_vs_reference(gpu, orc, ref, views_per_step):
    from paper_2412_03451_b200 import Optimizer
    P, cams, tg = _setup(orc, seed=5, n=6, n_views=4)
    oc = default_optim_config(orc)
    oc.enable_split = 0
    oc.lr_radii = 0.05
    oc.views_per_step = views_per_step
    oc.seed = 3
    r = RefOptimizer(ref, P, cams, tg, oc)
    dev = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    for it in range(10):
        assert dev.view_for_slot(it) == r.view_for_slot(it)
        lr, ld = r.step(), dev.step()
        assert abs(ld - lr) <= 1e-12 * abs(lr) + 1e-15, (it, ld, lr)
        _dev_state_equal(dev, r.state(), exact=False, rtol=1e-9)


def test_optimizer_run_with_split_vs_restatement(gpu, orc):
    """Optimizer::run semantics (maybe_split before each step) on a C1-like room."""
    from paper_2412_03451_b200 import Optimizer
    P, cams, tg = _setup(orc, seed=9, n=24, n_views=3, size=32)
    oc = default_optim_config(orc)
    oc.split_interval = 4
    oc.split_grad_threshold = 0.0  # every primitive with gradient splits at the boundary
    s = RestatedOptimizer(orc, OptimState.fresh(P), cams, tg, oc)
    dev = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    log = dev.run(9)
    assert len(log) == 9 and [r.iteration for r in log] == list(range(9))
    for it in range(9):
        s.maybe_split()
        lo = s.step()
        assert abs(log[it].loss - lo) <= 1e-9 * abs(lo) + 1e-12, it
        assert log[it].lam == dev.lambda_at(it)  # LossLogRow.lambda (optimizer.cpp:209-211)
    assert log[-1].primitive_count == s.st.planes.n > P.n
    _dev_state_equal(dev, s.st, exact=False, rtol=1e-7)


def _merge_dev(P, sc, **kw):
    from paper_2412_03451_b200 import OptimConfig, Optimizer
    oc = OptimConfig(**kw)
    dev = Optimizer(to_scene(P), [], oc, precision="fp64")
    return dev.merge_planes(sc)


def _merge_equal(dev_inst, o):
    assert len(dev_inst) == o["n"]
    for t, I in enumerate(dev_inst):
        assert I.member_indices == np.nonzero(o["instance_of"] == t)[0].tolist()
        assert np.array_equal(I.normal, o["normal"][t])
        assert I.offset == o["offset"][t] and I.area == o["area"][t]


@pytest.mark.parametrize("seed", [1, 88])
def test_merge_planes_bitwise_random(gpu, orc, seed):
    rng = np.random.default_rng(seed)
    n = 400
    P = Planes.empty(n)
    for i in range(n):
        q = rng.normal(size=4)
        P.center[i] = rng.uniform(-2, 2, 3)
        P.rotation[i] = q / np.sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]))
        P.radii[i] = rng.uniform(0.1, 0.6, 4)
        P.ids[i] = 5000 - 3 * i
    sc = (0.1, -0.2, 0.3)
    for use_adj in (True, False):
        o = orc.merge_planes(P, sc, 60.0, 0.3, 0.2, use_adj)
        _merge_equal(_merge_dev(P, sc, merge_normal_deg=60.0, merge_offset=0.3,
                                merge_adjacency=0.2, merge_use_adjacency=use_adj), o)


def test_merge_planes_bitwise_room(gpu, orc):
    from paper_2412_03451_b200 import scenes
    for name in ("c2", "c3"):
        s = scenes.load(name).scene
        P = Planes(s.center.copy(), s.rotation.copy(), s.radii.copy(), s.ids.copy())
        sc = P.center.mean(axis=0)
        o = orc.merge_planes(P, sc)
        d = _merge_dev(P, sc)
        _merge_equal(d, o)
        assert 1 < len(d) < P.n


# ---- init_from_depth (scene_init.cpp:70-104)
def _init_dev(cams, td, tn, n, seed, scale):
    from paper_2412_03451_b200 import ViewBatch
    vb = ViewBatch(precision="fp64")
    vb.set_views([to_view(c) for c in cams], td, tn)
    k = vb.init_from_depth(n, seed, scale)
    return vb.planes(), k


@pytest.fixture(scope="module")
def small_room(ref):
    from oracle.oracle import Camera, RefScenes
    rs = RefScenes()
    spec = (4.0, 4.0, 3.0, 1, 7)
    cams = list(rs.room_views(*spec, 40, 7, 48, 36))[:12]
    td, tn = rs.render_ground_truth(spec, (Camera * len(cams))(*cams))
    return cams, td, tn


@pytest.mark.parametrize("n,seed,scale", [(64, 7, 0.5), (500, 1, 0.5), (3000, 2, 0.25), (1, 3, 0.5),
                                          (30000, 4, 0.5)])
def test_init_from_depth_bitwise(gpu, orc, small_room, n, seed, scale):
    cams, td, tn = small_room
    want = orc.init_from_depth(cams, td, tn, n, seed, scale)
    got, k = _init_dev(cams, td, tn, n, seed, scale)
    assert k == want.n
    for a, b in [(got.center, want.center), (got.rotation, want.rotation), (got.radii, want.radii),
                 (got.ids, want.ids)]:
        assert np.array_equal(a, b)


def test_init_from_depth_errors(gpu, small_room):
    cams, td, tn = small_room
    with pytest.raises(ValueError):
        _init_dev(cams, td, tn, 0, 1, 0.5)
    with pytest.raises(RuntimeError, match="no valid depth pixels"):
        _init_dev(cams, np.zeros_like(td), tn, 5, 1, 0.5)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_init_from_depth_reproduces_committed_scenes(gpu, name):
    """The committed workload scenes were built by the reference's init_from_depth
    (scripts/make_scenes.py); the device rebuilds them bit for bit from targets it
    renders itself."""
    from paper_2412_03451_b200 import ViewBatch, scenes
    wl = scenes.load(name)
    vb = ViewBatch(precision="fp64")
    vb.set_views(list(wl.cams))
    vb.render_ground_truth(wl.faces)
    k = vb.init_from_depth(wl.scene.n, 7)
    got = vb.planes()
    assert k == wl.scene.n
    for a, b in [(got.center, wl.scene.center), (got.rotation, wl.scene.rotation),
                 (got.radii, wl.scene.radii), (got.ids, wl.scene.ids)]:
        assert np.array_equal(a, b)


def test_checkpoint_resume_continues_the_run(gpu, orc, tmp_path):
    """save_checkpoint / load_checkpoint (PSCK, dataio.cpp:250-330) of the device
    optimiser state: a resumed optimiser continues like the original run."""
    from paper_2412_03451_b200 import Optimizer, load_checkpoint, save_checkpoint
    P, cams, tg = _setup(orc, seed=5, n=6, n_views=4)
    oc = default_optim_config(orc)
    oc.lr_radii = 0.05
    oc.views_per_step = 2
    oc.split_interval = 3
    oc.split_grad_threshold = 0.0
    a = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    a.run(5)
    path = str(tmp_path / "run.psck")
    save_checkpoint(path, a.state(), 42)
    b = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    b.load_state(load_checkpoint(path, 42))
    la, lb = a.run(9), b.run(9)
    assert [r.iteration for r in la] == [r.iteration for r in lb] == [5, 6, 7, 8]
    for x, y in zip(la, lb):
        assert abs(x.loss - y.loss) <= 1e-12 * abs(x.loss) and x.primitive_count == y.primitive_count
    sa, sb = a.state(), b.state()
    np.testing.assert_allclose(sb.scene.center, sa.scene.center, rtol=1e-10, atol=1e-14)
    assert np.array_equal(sa.scene.ids, sb.scene.ids) and sa.next_id == sb.next_id


def test_sharded_step_equals_single_step(gpu, orc):
    """slot k of a step goes to rank k mod N and the gradients are summed
    before the identical Adam update. Two contexts stand in for two ranks one after
    the other (no cross-context waiting); the host sums their gradient buffers."""
    from paper_2412_03451_b200 import Optimizer
    P, cams, tg = _setup(orc, seed=5, n=40, n_views=6, size=32)
    oc = default_optim_config(orc)
    oc.views_per_step = 5
    oc.lr_radii = 0.05
    oc.seed = 11
    one = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    ranks = [Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64") for _ in range(2)]
    for it in range(6):
        want = one.step()
        parts = []
        for r, o in enumerate(ranks):
            o.step_local(r, 2)
            parts.append(o.read_grads())
        g = parts[0][0] + parts[1][0]
        loss = parts[0][1] + parts[1][1]
        got = []
        for o in ranks:
            o.set_gradients(g, loss)
            got.append(o.step_finish())
        assert got[0] == got[1] and abs(got[0] - want) <= 1e-12 * abs(want)
        assert ranks[0].params_checksum() == ranks[1].params_checksum()
        np.testing.assert_allclose(ranks[0].scene().center, one.scene().center, rtol=1e-10, atol=1e-15)


def test_deterministic_mode_bitwise_runs_and_resume(gpu, orc, tmp_path):
    """SURVEY App. B H3 / acceptance criterion 9: in deterministic mode repeated
    runs, and a run resumed from a PSCK checkpoint, are bitwise identical (splits
    included); the fixed-order sums agree with the atomic ones to rounding."""
    from paper_2412_03451_b200 import Optimizer, load_checkpoint, save_checkpoint
    P, cams, tg = _setup(orc, seed=5, n=30, n_views=5, size=32)
    oc = default_optim_config(orc)
    oc.views_per_step = 3
    oc.lr_radii = 0.05
    oc.split_interval = 7
    oc.split_grad_threshold = 0.0
    oc.seed = 3

    def make():
        o = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
        o.set_deterministic(True)
        return o

    a, b = make(), make()
    la, lb = a.run(20), b.run(20)
    assert [x.loss for x in la] == [x.loss for x in lb]
    sa, sb = a.state(), b.state()
    for x, y in [(sa.scene.center, sb.scene.center), (sa.scene.rotation, sb.scene.rotation),
                 (sa.scene.radii, sb.scene.radii), (sa.m, sb.m), (sa.v, sb.v)]:
        assert x.tobytes() == y.tobytes()
    assert sa.scene.n > P.n  # splits happened
    # resume through the checkpoint format
    c = make()
    c.run(10)
    save_checkpoint(str(tmp_path / "half.psck"), c.state(), 9)
    d = make()
    d.load_state(load_checkpoint(str(tmp_path / "half.psck"), 9))
    ld = d.run(20)
    assert [x.loss for x in ld] == [x.loss for x in la[10:]]
    sd = d.state()
    assert sd.scene.center.tobytes() == sa.scene.center.tobytes() and sd.m.tobytes() == sa.m.tobytes()
    # the atomic mode agrees to rounding
    e = Optimizer(to_scene(P), _views(orc, cams, tg), _ocfg(oc), precision="fp64")
    le = e.run(5)
    for x, y in zip(le, la[:5]):
        assert abs(x.loss - y.loss) <= 1e-12 * abs(y.loss)
