"""GPU: the synchronisation-free step and the 32-bit limits
(next #6).

psg_step never waits for the device: the bins and record blocks keep the sizes
earlier steps needed, and a step that does not fit aborts on the device
(k_bin_guard) and is replayed with exact sizes by the next call that reads
results, from the gradients and statistics of the window start. A step whose
(tile, plane) bin entries exceed the pair limit (2^31 - 1 by default: 32-bit CSR
offsets) is split into view groups. Contract: replayed and split steps give the
unsplit, unreplayed step's loss, per-view losses and maps, and gradients within
the run-to-run spread of fp64 atomics (1e-12 of max |g|).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    return True


@pytest.fixture(scope="module")
def c2():
    from paper_2412_03451_b200 import scenes
    return scenes.load("c2")


def _batch(wl, n=12, precision="fp64"):
    from paper_2412_03451_b200 import ViewBatch
    vb = ViewBatch(precision=precision)
    vb.set_scene(wl.scene)
    vb.set_views(list(wl.cams)[:n])
    vb.render_ground_truth(wl.faces)
    return vb


def _run(vb, ids, lam, maps=True):
    vb.zero_grads()
    vb.step(ids, lam, 1.0 / len(ids), write_maps=maps)
    vb.finalize()
    g, loss = vb.read_grads()
    return g, loss, vb.view_losses(len(ids))


def _close(a, b, what):
    ga, la, va = a
    gb, lb, vb_ = b
    assert abs(la - lb) <= 1e-12 * abs(lb), what
    np.testing.assert_allclose(va, vb_, rtol=1e-12, atol=0, err_msg=str(what))
    assert np.abs(ga - gb).max() <= 1e-12 * np.abs(gb).max(), what


def test_first_step_replays_then_runs_without_sync(gpu, c2):
    vb = _batch(c2)
    ids = np.arange(12)
    first = _run(vb, ids, 54.0)  # empty buffers: the step aborts and is replayed
    st = vb.stats()
    assert st["replays"] == 1 and st["zbound_violations"] == 0
    second = _run(vb, ids, 54.0)  # the buffers now fit: no replay
    assert vb.stats()["replays"] == 1
    _close(first, second, "replayed vs plain")
    # statistics count the replayed step once
    assert vb.stats()["views"] == 24 and vb.stats()["pairs"] == 2 * st["pairs"]


def test_window_of_several_steps_with_growth(gpu, c2):
    """Steps at lambda 300 size the buffers; a lambda-20 step in the same window
    outgrows them: the whole window (both steps, one accumulated gradient) replays."""
    a = _batch(c2)
    ids1, ids2 = np.arange(0, 6), np.arange(6, 12)
    for _ in range(2):  # size the buffers for the lambda-300 steps
        _run(a, ids1, 300.0, maps=False)
    r0 = a.stats()["replays"]
    a.zero_grads()
    a.step(ids1, 300.0, 0.5)
    a.step(ids2, 20.0, 0.5)  # more bin entries than the buffers hold: aborts
    a.finalize()
    ga, la = a.read_grads()
    assert a.stats()["replays"] == r0 + 1
    b = _batch(c2)
    b.set_deterministic(True)  # synchronous steps, exact sizes
    b.zero_grads()
    b.step(ids1, 300.0, 0.5)
    b.step(ids2, 20.0, 0.5)
    b.finalize()
    gb, lb = b.read_grads()
    assert abs(la - lb) <= 1e-12 * lb
    assert np.abs(ga - gb).max() <= 1e-12 * np.abs(gb).max()


@pytest.mark.parametrize("views_per_group", [5, 2, 1])
def test_pair_limit_splits_the_step(gpu, c2, views_per_group):
    ref = _batch(c2)
    ids = np.arange(12)
    per_view = []
    for k in ids:  # bin entries of each view alone
        before = ref.stats()["pairs"]
        _run(ref, [k], 54.0, maps=False)
        per_view.append(ref.stats()["pairs"] - before)
    want = _run(ref, ids, 54.0)
    _run(ref, ids, 54.0)
    maps_want = [ref.read_step_maps(k, c2.width, c2.height) for k in range(12)]
    pairs_per_step = sum(per_view)
    # a limit that fits about views_per_group views, and every single view
    limit = max(max(per_view), pairs_per_step * views_per_group // 12)
    assert pairs_per_step > limit  # the threshold is crossed
    vb = _batch(c2)
    vb.set_pair_limit(limit)
    got = _run(vb, ids, 54.0)
    _close(got, want, ("split", views_per_group))
    for k in range(12):
        for a, b in zip(vb.read_step_maps(k, c2.width, c2.height), maps_want[k]):
            assert np.array_equal(a, b), (views_per_group, k)
    assert vb.stats()["pairs"] == pairs_per_step  # the replayed window counted once
    # one view above the limit cannot be split
    vb.set_pair_limit(max(per_view) - 1)
    with pytest.raises(ValueError, match="32-bit limit"):
        _run(vb, [int(np.argmax(per_view))], 54.0)
    with pytest.raises(ValueError):
        vb.set_pair_limit(0)


def test_views_above_16_bit_pixel_coordinates_are_refused(gpu):
    from paper_2412_03451_b200 import CameraView, Renderer, Scene, ViewBatch
    big = CameraView(500.0, 500.0, 16000.0, 10.0, 32768, 20, np.eye(3), np.zeros(3))
    vb = ViewBatch(precision="fp64")
    with pytest.raises(ValueError, match="32767"):
        vb.set_views([big])
    r = Renderer(precision="fp64")
    sc = Scene(np.array([[0.0, 0.0, 2.0]]), np.array([[1.0, 0, 0, 0]]), np.full((1, 4), 0.5), np.zeros(1, np.int64))
    with pytest.raises(ValueError, match="32767"):
        r.render_view(big, sc, 300.0)
    ok = CameraView(500.0, 500.0, 16000.0, 10.0, 32767, 20, np.eye(3), np.zeros(3))
    vb.set_views([ok])  # the largest allowed side


def test_step_host_waits_for_earlier_steps_and_counts_streamed_targets(gpu, c2):
    """psg_step_host's copies wait for earlier work on the context stream,
    and the valid-pixel normalisers (renderer.cpp:328-334) come from the targets it
    is given: streaming targets with holes gives the loss of a context whose
    registered targets have the same holes."""
    n, npx = 6, c2.width * c2.height
    src = _batch(c2, n)
    td = src.pinned(n * npx * 4, np.float32)
    tn = src.pinned(n * npx * 12, np.float32)
    for k in range(n):
        a, b = src.get_targets(k)
        td[k * npx:(k + 1) * npx] = a
        tn[3 * k * npx:3 * (k + 1) * npx] = b
    td[::3] = 0.0  # invalid depth pixels
    tn[0:3 * npx:7] = 0.0
    want_ctx = _batch(c2, n)
    want_ctx.set_views(list(c2.cams)[:n], np.array(td), np.array(tn))
    want = _run(want_ctx, np.arange(n), 54.0, maps=False)
    vb = _batch(c2, n)  # registered targets without holes
    for _ in range(3):  # queue steps on the stream, then stream new targets in
        vb.zero_grads()
        vb.step(np.arange(n), 54.0, 1.0 / n)
    vb.zero_grads()
    vb.step_host(0, n, 54.0, td, tn, 1.0 / n, chunk_views=2)
    vb.finalize()
    g, loss = vb.read_grads()
    _close((g, loss, vb.view_losses(n)), want, "step_host")


def _opt(orc_scene, views, det, **kw):
    from paper_2412_03451_b200 import OptimConfig, Optimizer
    args = dict(views_per_step=3, seed=5, split_interval=7, split_grad_threshold=0.0, lr_radii=0.02)
    args.update(kw)
    o = Optimizer(orc_scene, views, OptimConfig(**args), precision="fp64")
    o.set_deterministic(det)
    return o


@pytest.mark.parametrize("pair_limit,det", [(None, True), ("tight", True), ("tight", False)])
def test_deferred_run_equals_step_loop(gpu, orc, pair_limit, det):
    """psg_optim_run enqueues blocks of iterations without host waits (Adam gated on
    the device) and reruns a halted iteration on the synchronous path. In
    deterministic mode it must equal, bitwise, the loop of psg_optim_maybe_split +
    psg_optim_step (optimizer.cpp:204-214) -- across split rounds, and with a pair
    limit that makes steps abort and replay as split view groups."""
    from _util import to_scene, to_view
    from paper_2412_03451_b200 import CameraView
    P = orc.random_scene(9, 40)
    views = []
    for k in range(5):
        cam = orc.make_view(48, 40, 30.0, True, 60 + k)
        td, tn = orc.fill_random_targets(cam, 60 + k)
        v = to_view(cam)
        views.append(CameraView(v.fx, v.fy, v.cx, v.cy, v.width, v.height, v.rot_wc, v.t_wc, td, tn))
    # the tight variant: 5-view steps, no split rounds (a split doubles every view's
    # bin entries), a limit of 1.5x the largest single view: every step splits
    kw = dict(views_per_step=5, enable_split=False) if pair_limit else {}
    a, b = _opt(to_scene(P), views, det, **kw), _opt(to_scene(P), views, det, **kw)
    if pair_limit:
        from paper_2412_03451_b200 import ViewBatch
        probe = ViewBatch(precision="fp64")
        probe.set_scene(to_scene(P))
        probe.set_views(views, np.concatenate([v.target_depth for v in views]),
                        np.concatenate([v.target_normal for v in views]))
        single = []
        for k in range(5):
            before = probe.stats()["pairs"]
            probe.zero_grads()
            probe.step([k], 7.4)
            probe.finalize()
            single.append(probe.stats()["pairs"] - before)
        limit = int(1.5 * max(single))
        assert limit < sum(single)
        for o in (a, b):
            o.set_pair_limit(limit)
    log = a.run(20)
    assert [r.iteration for r in log] == list(range(20))
    want = []
    for _ in range(20):
        b.maybe_split()
        want.append(b.step())
    sa, sb = a.state(), b.state()
    assert sa.scene.n == sb.scene.n and (pair_limit or sa.scene.n > 40)
    assert np.array_equal(sa.step, sb.step) and np.array_equal(sa.scene.ids, sb.scene.ids)
    pairs = ((sa.scene.center, sb.scene.center), (sa.scene.rotation, sb.scene.rotation),
             (sa.scene.radii, sb.scene.radii), (sa.m, sb.m), (sa.v, sb.v), (sa.radii_grad_sum, sb.radii_grad_sum))
    if det:  # deterministic mode is synchronous: the groups split inside the step, bitwise
        assert [r.loss for r in log] == want
        for x, y in pairs:
            assert x.tobytes() == y.tobytes()
    else:  # every deferred step aborts on the device, halts its block and reruns split
        np.testing.assert_allclose([r.loss for r in log], want, rtol=1e-12)
        for x, y in pairs:
            np.testing.assert_allclose(x, y, rtol=1e-9, atol=1e-9 * max(np.abs(y).max(), 1e-300))
        assert a.stats()["replays"] >= 20
