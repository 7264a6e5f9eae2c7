"""CPU, world_size 2 over gloo: the multi-GPU plumbing of bench.py (view dealing,
barrier, max-over-ranks timing) and the no-collective data path: each rank
renders its own views; only a scalar timing all-reduce crosses ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = bench.deal_views(10, world, rank)
    bench.barrier(dist)
    t = bench.max_over_ranks(dist, 1.0 + rank * 2.5, "cpu")
    # scene inputs are generated independently (and identically) on every rank
    import numpy as np
    import paper_2512_13796_b200 as nx
    s = nx.stump_like(1_000, log2_table=8)
    q.put((rank, views, t, float(np.abs(s.nexels).sum())))
    dist.destroy_process_group()


def test_two_rank_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(2):
        rank, views, t, chk = q.get(timeout=120)
        out[rank] = (views, t, chk)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v0, v1 = out[0][0], out[1][0]
    assert all(a != b for a, b in zip(v0, v1))              # disjoint views per step
    assert sorted(v0 + v1) == list(range(20))               # together: views 0..19, each once
    assert out[0][1] == out[1][1] == pytest.approx(3.5)     # max over ranks
    assert out[0][2] == out[1][2]                           # identical scene on each rank


def test_views_wrap_the_ring():
    sys.path.insert(0, ROOT)
    import bench
    v = bench.deal_views(300, 1, 0)
    assert v[255] == 255 and v[256] == 0
    allv = sorted(x for r in range(8) for x in bench.deal_views(32, 8, r))
    assert allv == list(range(256))


def test_frame_bytes_formula_matches_survey():
    """config 2 -> 4.32 GB/frame, config 1 -> 140.8 MB/frame."""
    sys.path.insert(0, ROOT)
    import bench
    b2 = bench.frame_bytes(400_000, 27_511_255, 1080, 1920, 2, 3_756_984)
    assert abs(b2 / 1e9 - 4.32) < 0.01
    b1 = bench.frame_bytes(10_000, 143_383, 256, 256, 2, 129_157)
    assert abs(b1 / 1e6 - 140.8) < 0.5


def test_image_bands_partition_the_rows():
    import paper_2512_13796_b200 as nx
    for H in (2160, 1080, 256, 100):
        for n in (1, 2, 3, 4, 8):
            bands = nx.image_bands(H, n)
            assert len(bands) == n
            y = 0
            for y0, rows in bands:
                assert y0 == min(y, H) and rows >= 0
                if rows:
                    assert y0 % 16 == 0
                y = y0 + rows
            assert y == H


def _dyn_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import time
    import torch.distributed as dist
    from paper_2512_13796_b200.views import DynamicDealer
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    dealer = DynamicDealer(100, store=store, start=7)
    got = []
    while (v := dealer.next()) is not None:
        got.append(v)
        time.sleep(0.001 * (1 + rank))  # rank 1 is slower: it should draw fewer views
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_dynamic_view_dealing_two_ranks():
    """Views pulled from one shared atomic counter (the store's add): every view of the
    run is rendered exactly once across the ranks, and the faster rank takes more."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dyn_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allv = sorted(out[0] + out[1])
    assert allv == sorted((7 + i) % 256 for i in range(100))
    assert len(out[0]) > len(out[1])


def test_view_groups_times_bands_cover_every_band_of_every_view():
    """Config 4 sharding: world 8 = 2 view groups x 4 bands; per step every view the
    groups render has all its bands rendered once, the bands partition the rows."""
    from paper_2512_13796_b200.views import ShardPlan
    world, H = 8, 2160
    plans = [ShardPlan(world, r, 4) for r in range(world)]
    for s in range(6):
        seen = {}
        for p in plans:
            v = p.views(6)[s]
            seen.setdefault(v, []).append(p.band_rows(H))
        assert len(seen) == 2  # two views per step (one per group)
        for v, bands in seen.items():
            bands.sort()
            assert bands[0][0] == 0 and sum(r for _, r in bands) == H
    with pytest.raises(ValueError):
        ShardPlan(8, 0, 3)
