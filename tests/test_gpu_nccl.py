"""GPU: the library's own NCCL path (psg_nccl_unique_id, psg_comm_init,
psg_allreduce_grads, psg_optim_step with a communicator and check_ranks), SURVEY.md
8e. Gradient semantics to match: Optimizer::step sums the per-view passes of the
step (optimizer.cpp:61-98), here split over ranks by slot k -> rank k mod N and
summed with one ncclAllReduce before the identical Adam update on every rank.

World size 1 runs on every GPU box: a one-rank communicator must leave the step
bit-identical to the communicator-free step (deterministic mode on both, so the
comparison is bitwise). The two-rank test runs whenever two GPUs are visible.
"""
import os
import tempfile

import numpy as np
import pytest

from _util import to_scene, to_view
from oracle.oracle import default_optim_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    return True


def _problem(orc, n_views=6):
    from paper_2412_03451_b200 import CameraView
    P = orc.random_scene(5, 60)
    views = []
    for k in range(n_views):
        cam = orc.make_view(40, 32, 24.0, True, 30 + k)
        td, tn = orc.fill_random_targets(cam, 30 + k)
        v = to_view(cam)
        views.append(CameraView(v.fx, v.fy, v.cx, v.cy, v.width, v.height, v.rot_wc, v.t_wc, td, tn))
    return P, views


def _cfg(orc, **kw):
    from paper_2412_03451_b200 import OptimConfig
    oc = default_optim_config(orc)
    o = OptimConfig(lr_center=oc.lr_center, lr_radii=0.05, lr_rotation=oc.lr_rotation,
                    views_per_step=5, seed=11, split_interval=3, split_grad_threshold=0.0)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def test_nccl_world1_step_bitwise_equal_to_no_comm(gpu, orc):
    from paper_2412_03451_b200 import Optimizer, nccl_unique_id
    P, views = _problem(orc)
    plain = Optimizer(to_scene(P), views, _cfg(orc), precision="fp64")
    comm = Optimizer(to_scene(P), views, _cfg(orc, check_ranks=True), precision="fp64")
    uid = nccl_unique_id()
    assert len(uid) == 128
    comm.comm_init(uid, 1, 0)
    for o in (plain, comm):
        o.set_deterministic(True)
    for it in range(7):  # crosses two split rounds (split_interval 3)
        kp, kc = plain.maybe_split(), comm.maybe_split()
        assert kp == kc
        lp, lc = plain.step(), comm.step()  # comm: local step -> ncclAllReduce -> finish -> rank check
        assert lp == lc, (it, lp, lc)
        assert plain.params_checksum() == comm.params_checksum()
    sp, sc = plain.state(), comm.state()
    assert sp.scene.center.tobytes() == sc.scene.center.tobytes()
    assert sp.m.tobytes() == sc.m.tobytes() and sp.v.tobytes() == sc.v.tobytes()


def test_allreduce_grads_world1_is_identity(gpu, orc):
    from paper_2412_03451_b200 import ViewBatch, nccl_unique_id
    P, views = _problem(orc, 3)
    vb = ViewBatch(precision="fp64")
    vb.set_scene(to_scene(P))
    vb.set_views(views, np.concatenate([v.target_depth for v in views]),
                 np.concatenate([v.target_normal for v in views]))
    with pytest.raises(ValueError, match="no communicator"):
        vb.allreduce_grads()
    vb.comm_init(nccl_unique_id(), 1, 0)
    vb.zero_grads()
    vb.step([0, 1, 2], 40.0, 1.0 / 3)
    g0, l0 = vb.read_grads()
    vb.allreduce_grads()
    g1, l1 = vb.read_grads()
    assert g0.tobytes() == g1.tobytes() and l0 == l1


def _rank_main(rank, world, port, out_dir, seed):
    """One rank of the two-GPU test: view-sharded Optimizer::step with NCCL."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from oracle.oracle import Oracle
    from paper_2412_03451_b200 import Optimizer
    from paper_2412_03451_b200.dist import nccl_bootstrap
    orc = Oracle("orc")
    P, views = _problem(orc)
    # no split rounds: splits make exactly coplanar children whose (z, prim) order at
    # a pixel is decided by 1-ulp differences, and the two-rank
    # gradient sum rounds differently from the one-rank sum
    o = Optimizer(to_scene(P), views, _cfg(orc, check_ranks=True, enable_split=False), device=rank,
                  precision="fp64")
    o.set_deterministic(True)
    nccl_bootstrap(o, rank, world)
    losses = []
    for _ in range(7):
        o.maybe_split()
        losses.append(o.step())
    s = o.state()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), losses=np.array(losses), center=s.scene.center,
             m=s.m, checksum=np.array([o.params_checksum()], np.uint64))
    dist.barrier(device_ids=[rank])
    dist.destroy_process_group()


def test_two_gpu_sharded_optimizer_matches_single_gpu(gpu, orc):
    import socket

    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 visible GPUs (this pool's boxes expose one)")
    from paper_2412_03451_b200 import Optimizer
    P, views = _problem(orc)
    one = Optimizer(to_scene(P), views, _cfg(orc, enable_split=False), precision="fp64")
    want = []
    for _ in range(7):
        one.maybe_split()
        want.append(one.step())
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(2, port, d, 0), nprocs=2, join=True)
        r0, r1 = (np.load(os.path.join(d, f"rank{r}.npz")) for r in (0, 1))
        assert np.array_equal(r0["losses"], r1["losses"]) and r0["checksum"][0] == r1["checksum"][0]
        np.testing.assert_allclose(r0["losses"], want, rtol=1e-12)
        np.testing.assert_allclose(r0["center"], one.scene().center, rtol=1e-9, atol=1e-15)
