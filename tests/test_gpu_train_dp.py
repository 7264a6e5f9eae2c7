"""GPU, world size 2 (two processes on one GPU, gloo for the gradient all-reduce):
the data-parallel training iteration (train_dp.DataParallelStep). The replicas stay
bit-identical, and the averaged gradient of an iteration is exactly the mean of the two
views' single-process gradients (the backward is bit-reproducible)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W, H, N = 160, 120, 20_000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(world, rank):
    import torch
    import paper_2512_13796_b200 as nx
    from paper_2512_13796_b200.train_dp import DataParallelStep, device_view
    scene = nx.stump_like(N, log2_table=14)
    target = nx.stump_like(N, log2_table=14, grid_init=1e-1)
    r = nx.Renderer(0)
    cams = {v: nx.ring_camera(v, 256, W, H) for v in range(0, 256, 16)}
    ts = r.upload(target)
    tf = r.frame()
    gt = {}
    for v, c in cams.items():
        r.render(ts, c, tf)
        r.synchronize()
        gt[v] = device_view(tf.view().final_img, W * H * 3, torch.float32, torch.device("cuda", 0)).double()
    tf.close()
    ts.close()
    ds = r.upload(scene)
    return nx, r, scene, ds, cams, gt, DataParallelStep


def _dp_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2512_13796_b200.train_dp import rank_views
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, r, scene, ds, cams, gt, DataParallelStep = _setup(world, rank)
    step = DataParallelStep(r, ds, scene, cams, gt, dist=dist)
    views = rank_views(len(cams), 3, world, rank)
    vlist = sorted(cams)
    first = None
    for i, vi in enumerate(views):
        step.step(vlist[vi])
        r.synchronize()
        if i == 0:
            first = [t.cpu().numpy().copy() for t in step.grads]
    params = r.download_scene(ds, scene.field)
    q.put((rank, [vlist[v] for v in views], first, params, step.blend.cpu().numpy()))
    step.close()
    dist.barrier()
    dist.destroy_process_group()


def _single_worker(views, q):
    sys.path.insert(0, ROOT)
    nx, r, scene, ds, cams, gt, DataParallelStep = _setup(1, 0)
    out = []
    for v in views:  # gradients of each view from the same (un-updated) scene
        step = DataParallelStep(r, ds, scene, cams, gt)
        step.step(v)
        r.synchronize()
        out.append([t.cpu().numpy().copy() for t in step.grads])
        step.close()
        ds.close()
        ds = r.upload(scene)
    q.put(out)


def test_data_parallel_step_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((x[0], x[1:]) for x in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (v0, g0, p0, b0), (v1, g1, p1, b1) = res[0], res[1]
    assert v0[0] != v1[0]  # the ranks trained on different views
    for a, b in zip(g0, g1):  # the all-reduced gradient is the same on both ranks
        assert np.array_equal(a, b)
    for a, b in zip(p0, p1):  # the replicas stay bit-identical
        assert np.array_equal(a, b)
    assert np.array_equal(b0, b1)
    # iteration 1's averaged gradient = the mean of the two views' single-process gradients
    q2 = ctx.Queue()
    p = ctx.Process(target=_single_worker, args=([v0[0], v1[0]], q2))
    p.start()
    ga, gb = q2.get(timeout=600)
    p.join(timeout=120)
    for dp, a, b in zip(g0, ga, gb):
        assert np.array_equal(dp, (a + b) * 0.5)
    assert np.abs(g0[0]).max() > 0
