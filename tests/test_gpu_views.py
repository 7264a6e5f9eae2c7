"""GPU: the batched multi-view entry (nx_render_views) and per-context isolation —
two contexts rendering concurrently from two host threads on one device (each with its
own scene copy, lists and frames, as the per-GPU processes of the multi-GPU run have)
give the same bits as one context rendering alone."""
import threading

import numpy as np
import pytest

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200.views import DynamicDealer, render_dealt

pytestmark = pytest.mark.gpu

W, H = 320, 240


@pytest.fixture(scope="module")
def scene():
    return nx.stump_like(40_000, grid_init=1e-1)


def _alone(scene, views):
    r = nx.Renderer(0)
    ds = r.upload(scene)
    out = {}
    for v in views:
        f = r.frame()
        r.render(ds, nx.ring_camera(v, 256, W, H), f)
        g = f.download()
        out[v] = (g.ids.copy(), g.final_img.copy())
        f.close()
    ds.close()
    r.close()
    return out


def test_render_views_matches_single_renders(scene):
    views = [3, 50, 97, 140, 201, 255]
    ref = _alone(scene, views)
    r = nx.Renderer(0)
    ds = r.upload(scene)
    frames = [r.frame() for _ in range(len(views))]
    r.render_views(ds, [nx.ring_camera(v, 256, W, H) for v in views], frames)
    for v, f in zip(views, frames):
        g = f.download()
        assert np.array_equal(g.ids, ref[v][0]) and np.array_equal(g.final_img, ref[v][1]), v
    # fewer frames than views: the last len(frames) views survive in rotation
    r.render_views(ds, [nx.ring_camera(v, 256, W, H) for v in views], frames[:2])
    for v, f in zip(views[-2:], (frames[0], frames[1])):
        g = f.download()
        assert np.array_equal(g.final_img, ref[v][1]), v


def test_two_contexts_concurrently_are_isolated(scene):
    views = {0: [0, 16, 32, 48, 64, 80], 1: [8, 24, 40, 56, 72, 88]}
    ref = _alone(scene, views[0] + views[1])
    got, errors = {}, []

    def worker(k):
        try:
            r = nx.Renderer(0)
            ds = r.upload(scene)
            frames = [r.frame() for _ in range(3)]
            # the dealer hands out indices into this worker's view list
            dealer = DynamicDealer(len(views[k]), n_views=len(views[k]))
            cams = {i: nx.ring_camera(v, 256, W, H) for i, v in enumerate(views[k])}
            order = render_dealt(r, ds, cams, frames, dealer)
            assert order == list(range(len(views[k])))
            out = {}
            for n, i in enumerate(order):
                if n >= len(order) - 3:  # the frames still holding their views
                    g = frames[n % 3].download()
                    out[views[k][i]] = (g.ids.copy(), g.final_img.copy())
            got[k] = out
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for k in (0, 1):
        assert len(got[k]) == 3
        for v, (ids, fin) in got[k].items():
            assert np.array_equal(ids, ref[v][0]) and np.array_equal(fin, ref[v][1]), (k, v)

