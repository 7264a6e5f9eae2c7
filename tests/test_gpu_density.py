"""GPU: density control on the device scene — densify_split and prune
(density.cpp:102-177) with the optimizer rows following (adam_remap_rows,
adam.cpp:24-42) — against the reference's own functions: the same split parents
(from the same uniform draws), children geometry, survivor order, and the Adam step
after the remap."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi

pytestmark = pytest.mark.gpu

WIDTH = [3, 4, 2, 1, 2, 3, 45]
COLS = [slice(0, 3), slice(3, 7), slice(7, 9), slice(9, 10), slice(10, 12), slice(12, 15), slice(15, 60)]


def dev(a, dtype=torch.float64):
    return torch.tensor(np.ascontiguousarray(a).reshape(-1), dtype=dtype, device="cuda")


@pytest.mark.parametrize("n0", [3_000, 400_000])  # the latter: BASELINE config-5 scale (40K splits)
def test_densify_then_prune_match_reference(renderer, reference, n0):
    scene = nx.stump_like(n0, log2_table=10, grid_init=1e-1)
    n = scene.nexels.shape[0]
    budget = n + n // 10 + n // 30
    rng = np.random.default_rng(4)
    errors = rng.random(n) * (rng.random(n) > 0.3)  # some zero errors: never sampled
    ref_nex, ref_map, ref_splits, uniforms = reference.densify_split(scene.nexels, errors, budget, 0.1, 77)
    assert ref_splits == n // 10 and ref_nex.shape[0] == n + n // 10

    ds = renderer.upload(scene)
    opt = C.c_void_p()
    renderer._check(renderer.lib.nx_optimizer_create(renderer.ctx, ds.handle, C.byref(opt)))
    # one Adam step so that the remapped moments are non-trivial
    g0 = rng.standard_normal((n, 60))
    f = scene.field
    gf = [np.zeros(np.size(a)) for a in (f.table, f.w1, f.w2, f.w3)]
    tg = [dev(g0)] + [dev(a) for a in gf]
    cfg = (_abi.nx_adam_config * 11)(*[_abi.nx_adam_config(1e-3 if i < 7 else 0.0, 0.9, 0.999, 1e-8)
                                       for i in range(11)])
    gg = _abi.nx_grads(*(t.data_ptr() for t in tg))
    torch.cuda.synchronize()
    renderer._check(renderer.lib.nx_optimizer_step(renderer.ctx, opt, ds.handle, C.byref(gg), cfg, None))
    renderer.synchronize()
    # the same step on the host (reference adam_step per group)
    ref_params = renderer.download_scene(ds, f)[0]
    states = {}
    host = scene.nexels.copy()
    for gi in range(7):
        p = np.ascontiguousarray(host[:, COLS[gi]]).reshape(-1)
        m, v = np.zeros(p.size), np.zeros(p.size)
        reference.adam_step(m, v, 0, (1e-3, 0.9, 0.999, 1e-8), p, np.ascontiguousarray(g0[:, COLS[gi]]).reshape(-1))
        states[gi] = (m, v)
        host[:, COLS[gi]] = p.reshape(n, -1)
    assert np.allclose(ref_params[:, :12], host[:, :12], rtol=1e-12, atol=1e-15)

    # ---- densify_split with the reference's draws
    ref_nex, ref_map, ref_splits, uniforms = reference.densify_split(ref_params, errors, budget, 0.1, 77)
    n2o = torch.zeros(budget, dtype=torch.int32, device="cuda")
    n_out, sc = C.c_int64(), C.c_int64()
    e_t, u_t = dev(errors), dev(uniforms)
    renderer._check(renderer.lib.nx_scene_densify_split(renderer.ctx, ds.handle, opt, C.c_void_p(e_t.data_ptr()),
                                                        C.c_void_p(u_t.data_ptr()), budget, 0.1,
                                                        C.c_void_p(n2o.data_ptr()), C.byref(n_out), C.byref(sc)))
    assert (n_out.value, sc.value) == (ref_nex.shape[0], ref_splits)
    assert np.array_equal(n2o[: n_out.value].cpu().numpy(), ref_map)
    ds.n = n_out.value
    got = renderer.download_scene(ds, f)[0]
    assert np.allclose(got[:, :12], ref_nex[:, :12], rtol=1e-12, atol=1e-14)
    assert np.allclose(got[:, 12:], ref_nex[:, 12:], rtol=1e-6, atol=1e-7)  # SH stored fp32

    # ---- prune
    ref_pruned, ref_pmap = reference.prune(ref_nex, 0.55)
    assert 0 < ref_pruned.shape[0] < ref_nex.shape[0]
    pmap = torch.zeros(n_out.value, dtype=torch.int32, device="cuda")
    n2 = C.c_int64()
    renderer._check(renderer.lib.nx_scene_prune(renderer.ctx, ds.handle, opt, 0.55, C.c_void_p(pmap.data_ptr()),
                                                C.byref(n2)))
    assert n2.value == ref_pruned.shape[0]
    assert np.array_equal(pmap[: n2.value].cpu().numpy(), ref_pmap)
    ds.n = n2.value
    got = renderer.download_scene(ds, f)[0]
    assert np.allclose(got[:, :12], ref_pruned[:, :12], rtol=1e-12, atol=1e-14)

    # ---- the moments followed the rows: a second Adam step agrees with the reference's
    g1 = rng.standard_normal((n2.value, 60))
    tg = [dev(g1)] + [dev(a) for a in gf]
    gg = _abi.nx_grads(*(t.data_ptr() for t in tg))
    torch.cuda.synchronize()
    renderer._check(renderer.lib.nx_optimizer_step(renderer.ctx, opt, ds.handle, C.byref(gg), cfg, None))
    renderer.synchronize()
    after = renderer.download_scene(ds, f)[0]
    host = ref_pruned.copy()
    for gi in range(7):
        m, v = states[gi]
        m, v = reference.adam_remap_rows(m, v, ref_map, WIDTH[gi])
        m, v = reference.adam_remap_rows(m, v, ref_pmap, WIDTH[gi])
        p = np.ascontiguousarray(host[:, COLS[gi]]).reshape(-1)
        reference.adam_step(m, v, 1, (1e-3, 0.9, 0.999, 1e-8), p, np.ascontiguousarray(g1[:, COLS[gi]]).reshape(-1))
        host[:, COLS[gi]] = p.reshape(n2.value, -1)
    assert np.allclose(after[:, :12], host[:, :12], rtol=1e-11, atol=1e-14)
    renderer.lib.nx_optimizer_destroy(opt)


def test_density_control_on_an_empty_scene(renderer, reference):
    """densify_split and prune of an empty scene: nothing to split or keep, like the
    reference's (density.cpp:102-177)."""
    base = nx.stump_like(500, log2_table=10, grid_init=1e-1)
    scene = nx.Scene(np.zeros((0, 60)), base.field, base.settings)
    ref_nex, ref_map, ref_splits, _ = reference.densify_split(scene.nexels, np.zeros(0), 16, 0.1, 77)
    ref_pruned, _ = reference.prune(scene.nexels, 0.5)
    assert ref_nex.shape[0] == 0 and ref_splits == 0 and ref_pruned.shape[0] == 0
    ds = renderer.upload(scene)
    opt = renderer.optimizer(ds)
    n2o = torch.zeros(16, dtype=torch.int32, device="cuda")
    e_t = torch.zeros(1, dtype=torch.float64, device="cuda")
    u_t = torch.zeros(1, dtype=torch.float64, device="cuda")
    n_out, sc = C.c_int64(-1), C.c_int64(-1)
    renderer._check(renderer.lib.nx_scene_densify_split(renderer.ctx, ds.handle, opt.handle,
                                                        C.c_void_p(e_t.data_ptr()), C.c_void_p(u_t.data_ptr()), 16,
                                                        0.1, C.c_void_p(n2o.data_ptr()), C.byref(n_out),
                                                        C.byref(sc)))
    assert (n_out.value, sc.value) == (0, 0)
    pmap = torch.zeros(1, dtype=torch.int32, device="cuda")
    n2 = C.c_int64(-1)
    renderer._check(renderer.lib.nx_scene_prune(renderer.ctx, ds.handle, opt.handle, 0.5,
                                                C.c_void_p(pmap.data_ptr()), C.byref(n2)))
    assert n2.value == 0
