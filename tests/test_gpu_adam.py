"""GPU: Adam on the device scene (nx_optimizer_step) against the reference's
adam_step (adam.cpp:9-22) applied group by group like the trainer
(trainer.cpp:238-323): the same parameters, gradients and AdamConfigs for three
steps. Geometry is fp64 on both sides; SH / table / MLP weights are fp32 on the
device (the checkpoint precision), so those agree to fp32 rounding."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi

pytestmark = pytest.mark.gpu

# (group, column slice of the 60-value Nexel row or field array)
GEOM = {0: slice(0, 3), 1: slice(3, 7), 2: slice(7, 9), 3: slice(9, 10), 4: slice(10, 12), 5: slice(12, 15),
        6: slice(15, 60)}


def test_adam_steps_match_reference(renderer, reference):
    scene = nx.stump_like(2_000, log2_table=10, grid_init=1e-1)
    ds = renderer.upload(scene)
    opt = C.c_void_p()
    renderer._check(renderer.lib.nx_optimizer_create(renderer.ctx, ds.handle, C.byref(opt)))
    rng = np.random.default_rng(3)
    cfgs = [(1.6e-4 * 8.0, 0.9, 0.999, 1e-15), (1e-3, 0.9, 0.999, 1e-15), (5e-3, 0.9, 0.999, 1e-15),
            (5e-2, 0.9, 0.999, 1e-15), (1e-2, 0.9, 0.999, 1e-15), (2.5e-3, 0.9, 0.999, 1e-15),
            (1.25e-4, 0.9, 0.999, 1e-15), (1e-2, 0.9, 0.999, 1e-15), (1e-3, 0.9, 0.999, 1e-15),
            (1e-3, 0.9, 0.999, 1e-15), (-1.0, 0.9, 0.999, 1e-15)]  # w3 frozen: lr < 0 skips the group
    ccfg = (_abi.nx_adam_config * 11)(*[_abi.nx_adam_config(*c) for c in cfgs])
    f = scene.field
    ref_p = [scene.nexels.copy(), f.table.copy(), f.w1.copy(), f.w2.copy(), f.w3.copy()]
    # reference AdamStates per group (AoS order of gather_group, trainer.cpp:126-142)
    ref_state = {}
    for step in range(3):
        g_prims = rng.standard_normal((2_000, 60))
        g_f = [rng.standard_normal(np.size(a)) for a in (f.table, f.w1, f.w2, f.w3)]
        dev = [torch.tensor(a.reshape(-1), dtype=torch.float64, device="cuda") for a in (g_prims, *g_f)]
        gg = _abi.nx_grads(*(t.data_ptr() for t in dev))
        torch.cuda.synchronize()
        renderer._check(renderer.lib.nx_optimizer_step(renderer.ctx, opt, ds.handle, C.byref(gg), ccfg, None))
        renderer.synchronize()
        for gi in range(11):
            if cfgs[gi][0] < 0.0:
                continue
            if gi < 7:
                params = np.ascontiguousarray(ref_p[0][:, GEOM[gi]]).reshape(-1)
                grads = np.ascontiguousarray(g_prims[:, GEOM[gi]]).reshape(-1)
            else:
                params, grads = ref_p[gi - 6], g_f[gi - 7]
            m, v, st = ref_state.get(gi, (np.zeros(params.size), np.zeros(params.size), 0))
            st = reference.adam_step(m, v, st, cfgs[gi], params, grads)
            ref_state[gi] = (m, v, st)
            if gi < 7:
                ref_p[0][:, GEOM[gi]] = params.reshape(2_000, -1)
    steps = (C.c_int64 * 11)()
    renderer.lib.nx_optimizer_steps(opt, steps)
    assert list(steps) == [3] * 10 + [0]
    got = renderer.download_scene(ds, f)
    # geometry (fp64): exact up to the last ulp; fp32-stored groups: fp32 rounding
    assert np.allclose(got[0][:, :12], ref_p[0][:, :12], rtol=1e-12, atol=1e-15)
    assert np.allclose(got[0][:, 12:], ref_p[0][:, 12:], rtol=2e-6, atol=1e-6)
    for a, b in zip(got[1:], ref_p[1:]):
        assert np.allclose(a, b, rtol=2e-6, atol=1e-6)
    assert not np.allclose(got[0][:, :3], scene.nexels[:, :3])  # the positions moved
    renderer.lib.nx_optimizer_destroy(opt)


@pytest.mark.parametrize("n,log2", [(500, 8), (400_000, 20)])  # the latter: BASELINE config-5 scale
def test_fp64_masters_track_the_reference_exactly(renderer, reference, n, log2):
    """The fp32-stored groups (SH, table, MLP) are stepped on the optimizer's fp64 masters:
    read back with nx_optimizer_download they agree with the reference's fp64 adam_step to
    fp64 rounding, not just fp32 (the scene keeps their fp32 rounding for rendering)."""
    scene = nx.stump_like(n, log2_table=log2, grid_init=1e-1)
    ds = renderer.upload(scene)
    opt = renderer.optimizer(ds)
    f = scene.field
    init = {5: scene.nexels[:, 12:15], 6: scene.nexels[:, 15:60], 7: f.table, 8: f.w1, 9: f.w2, 10: f.w3}
    # seed the masters exactly (here the values are fp32-representable anyway)
    for gi, vals in init.items():
        opt.set_params(gi, vals)
    cfgs = [(1e-3, 0.9, 0.999, 1e-8)] * 11
    rng = np.random.default_rng(7)
    ref = {gi: np.ascontiguousarray(v, dtype=np.float64).reshape(-1).copy() for gi, v in init.items()}
    state = {}
    for _ in range(4):
        g_prims = rng.standard_normal((n, 60))
        g_f = [rng.standard_normal(np.size(a)) for a in (f.table, f.w1, f.w2, f.w3)]
        dev = [torch.tensor(a.reshape(-1), dtype=torch.float64, device="cuda") for a in (g_prims, *g_f)]
        torch.cuda.synchronize()
        opt.step([t.data_ptr() for t in dev], cfgs)
        renderer.synchronize()
        grads = {5: g_prims[:, 12:15], 6: g_prims[:, 15:60], 7: g_f[0], 8: g_f[1], 9: g_f[2], 10: g_f[3]}
        for gi in ref:
            gr = np.ascontiguousarray(grads[gi]).reshape(-1)
            m, v, st = state.get(gi, (np.zeros(gr.size), np.zeros(gr.size), 0))
            state[gi] = (m, v, reference.adam_step(m, v, st, cfgs[gi], ref[gi], gr))
    assert opt.steps() == [4] * 11
    for gi, want in ref.items():
        assert opt.size(gi) == want.size
        got, m, v = opt.download(gi)
        # fp64 on both sides (the device contracts some products into FMAs): a few ulp of
        # each array's scale
        for a, b in ((got, want), (m, state[gi][0]), (v, state[gi][1])):
            assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max(), gi
    opt.close()


def test_pixel_error_matches_the_trainer(renderer):
    """nx_pixel_error: err[p] = sum_c |final - gt| / 3 (trainer.cpp:288-295)."""
    scene = nx.stump_like(3_000, log2_table=10, grid_init=1e-1)
    cam = nx.ring_camera(5, 256, 96, 64)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    renderer.render(ds, cam, fr)
    fin = fr.download(["final_img"]).final_img.astype(np.float64)
    gt = np.random.default_rng(1).random(fin.size)
    gt_d = torch.tensor(gt, dtype=torch.float64, device="cuda")
    err_d = torch.empty(cam.width * cam.height, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    renderer.pixel_error(fr, gt_d.data_ptr(), err_d.data_ptr())
    renderer.synchronize()
    want = np.abs(fin - gt).reshape(-1, 3).sum(axis=1) / 3.0
    assert np.allclose(err_d.cpu().numpy(), want, rtol=1e-15, atol=1e-15)


def test_adam_on_an_empty_scene(renderer):
    """No primitives: the primitive groups are empty but still count the step like the
    reference's adam_step (adam.cpp:11-12 increments state.step whatever the count), the
    field groups step (zero gradients leave them unchanged) and nothing faults."""
    base = nx.stump_like(1_000, log2_table=10, grid_init=1e-1)
    scene = nx.Scene(np.zeros((0, 60)), base.field, base.settings)
    ds = renderer.upload(scene)
    opt = renderer.optimizer(ds)
    assert opt.size(0) == 0
    before = opt.download(8)[0]
    grads = [torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
             for n in (0, base.field.grid.param_count(), base.field.w1.size, base.field.w2.size, base.field.w3.size)]
    torch.cuda.synchronize()
    opt.step([t.data_ptr() for t in grads], [(1e-3, 0.9, 0.999, 1e-8)] * 11)
    renderer.synchronize()
    assert opt.steps() == [1] * 11
    assert np.array_equal(opt.download(8)[0], before)


def test_bad_primitive_after_a_parameter_change(renderer):
    """The reference activates every primitive on every render (renderer.cpp:38,
    primitive.cpp:47-63): a parameter change that makes a primitive non-finite or its
    quaternion degenerate fails the next render with bad-primitive and the first failing
    id; fixing the values clears it."""
    scene = nx.stump_like(2_000, log2_table=10)
    cam = nx.ring_camera(3, 256, 64, 48)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    renderer.render(ds, cam, fr)
    opt = renderer.optimizer(ds)
    pos, _, _ = opt.download(0)
    bad = pos.copy()
    bad[3 * 41 + 1] = np.nan
    bad[3 * 1500] = np.inf
    opt.set_params(0, bad)
    with pytest.raises(nx.NexelError) as e:
        renderer.render(ds, cam, fr)
    assert e.value.code == "bad-primitive" and "non-finite position in primitive 41" in str(e.value)
    q, _, _ = opt.download(1)
    opt.set_params(0, pos)
    q0 = q.copy()
    q0[4 * 7:4 * 8] = 0.0
    opt.set_params(1, q0)
    with pytest.raises(nx.NexelError) as e:
        renderer.render(ds, cam, fr)
    assert e.value.code == "bad-primitive" and "degenerate quaternion in primitive 7" in str(e.value)
    opt.set_params(1, q)
    renderer.render(ds, cam, fr)  # valid again
    opt.close()
