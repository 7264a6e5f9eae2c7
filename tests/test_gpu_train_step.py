"""GPU: a few whole training iterations (trainer.cpp:262-323 without density
control) on the device — render, losses_backward, per-pixel error, render_backward,
Adam over the 11 groups — against the same iterations composed from the
reference's own functions on the host. The loss terms of every iteration must
agree (the trajectories drift apart only by the fp32 storage of SH / table / MLP
weights on the device)."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import LossWeights, SceneGrads, UpstreamGrads, _abi

pytestmark = pytest.mark.gpu

GEOM = {0: slice(0, 3), 1: slice(3, 7), 2: slice(7, 9), 3: slice(9, 10), 4: slice(10, 12), 5: slice(12, 15),
        6: slice(15, 60)}


def lrs(extent):  # trainer.hpp:30-42 defaults, trainer.cpp:240-250
    return [(1.6e-4 * extent, 1e-15), (1e-3, 1e-8), (5e-3, 1e-8), (5e-2, 1e-8), (2e-3, 1e-8), (2.5e-3, 1e-8),
            (1.25e-4, 1e-8), (1e-2, 1e-8), (1e-3, 1e-8), (1e-3, 1e-8), (1e-3, 1e-8)]


def test_training_iterations_match_reference(renderer, reference):
    target = nx.stump_like(3_000, log2_table=12, grid_init=1e-1)
    scene = nx.stump_like(3_000, log2_table=12, grid_init=1e-4)
    cam = nx.ring_camera(12, 256, 96, 64)
    gt = reference.render(target, cam).final_img.copy()
    w = LossWeights()
    cfgs = lrs(scene.extent)
    iters = 4

    # ---- reference: the trainer's iteration from the reference's own functions
    ref_scene = nx.Scene(scene.nexels.copy(), nx.TextureField(scene.field.grid, scene.field.table.copy(),
                                                              scene.field.w1.copy(), scene.field.w2.copy(),
                                                              scene.field.w3.copy(), scene.field.n_hidden),
                         scene.settings, scene.extent)
    states = {}
    ref_losses = []
    K = scene.settings.top_k
    for it in range(iters):
        fb = reference.render(ref_scene, cam)
        terms, df, dw, dt, gp, gtab = reference.losses_backward(
            ref_scene, cam.width, cam.height, K, fb.ids, fb.weights, fb.texture, fb.final_img, gt,
            [w.dssim, w.alpha, w.texture, w.opacity, w.grid])
        ref_losses.append(terms)
        err = np.abs(fb.final_img - gt).reshape(-1, 3).mean(axis=1)
        p, tab, w1, w2, w3, be = reference.render_backward(ref_scene, cam, df, dw, dt, err)
        gp = gp + p
        gtab = gtab + tab
        gfield = [gtab, w1, w2, w3]
        for gi in range(11):
            lr, eps = cfgs[gi]
            if gi < 7:
                params = np.ascontiguousarray(ref_scene.nexels[:, GEOM[gi]]).reshape(-1)
                grads = np.ascontiguousarray(gp[:, GEOM[gi]]).reshape(-1)
            else:
                params = [ref_scene.field.table, ref_scene.field.w1, ref_scene.field.w2, ref_scene.field.w3][gi - 7]
                grads = gfield[gi - 7]
            m, v, st = states.get(gi, (np.zeros(params.size), np.zeros(params.size), 0))
            states[gi] = (m, v, reference.adam_step(m, v, st, (lr, 0.9, 0.999, eps), params, grads))
            if gi < 7:
                ref_scene.nexels[:, GEOM[gi]] = params.reshape(ref_scene.nexels.shape[0], -1)

    # ---- device: the same iterations through the C-ABI
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    opt = C.c_void_p()
    renderer._check(renderer.lib.nx_optimizer_create(renderer.ctx, ds.handle, C.byref(opt)))
    acfg = (_abi.nx_adam_config * 11)(*[_abi.nx_adam_config(lr, 0.9, 0.999, eps) for lr, eps in cfgs])
    dev = torch.device("cuda")
    for it in range(iters):
        renderer.render(ds, cam, fr)
        g = SceneGrads.allocate(scene)
        terms, df, dw, dt = renderer.losses_backward(ds, fr, gt, w, g)
        fin = fr.download(["final_img"]).final_img.astype(np.float64)
        err = np.abs(fin - gt).reshape(-1, 3).mean(axis=1)
        renderer.render_backward(ds, cam, fr, UpstreamGrads(df, dw, dt), g, err, np.zeros(scene.nexels.shape[0]))
        tg = [torch.tensor(a.reshape(-1), dtype=torch.float64, device=dev) for a in (g.prims, g.table, g.w1, g.w2,
                                                                                    g.w3)]
        gg = _abi.nx_grads(*(t.data_ptr() for t in tg))
        torch.cuda.synchronize()
        renderer._check(renderer.lib.nx_optimizer_step(renderer.ctx, opt, ds.handle, C.byref(gg), acfg, None))
        renderer.synchronize()
        for k in ("l1", "dssim", "texture", "alpha", "opacity", "grid", "total"):
            assert terms[k] == pytest.approx(ref_losses[it][k], rel=1e-4, abs=1e-9), (it, k)
    renderer.lib.nx_optimizer_destroy(opt)
    print([round(t["total"], 6) for t in ref_losses])
