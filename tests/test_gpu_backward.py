"""GPU parity of render_backward (renderer.cpp:251-401) against the reference
compiled in place (oracle/_ref): primitive gradients (mu, quat, log_scale,
opacity_raw, gamma_raw, sh), field gradients (hash table, w1, w2, w3) and the
blended-error accumulator, for the same scene, camera and seeded upstream
gradients. Cases follow the reference's gradient tests (proj/tests/
test_renderer.cpp:355-412, acceptance.cpp:48-88: random scenes, K = 0..4,
settings ablations) plus stump_like scenes at the BASELINE.json shapes.
"""
import numpy as np
import pytest

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import NexelError, SceneGrads, UpstreamGrads
from parity import GRAD_TOL_TC, compare_grads

pytestmark = pytest.mark.gpu


def upstream(cam, K, seed, parts=("final", "weights", "texture")):
    rng = np.random.default_rng(seed)
    npix = cam.width * cam.height
    return UpstreamGrads(
        d_final=rng.standard_normal(npix * 3) if "final" in parts else None,
        d_weights=rng.standard_normal(npix * K) if "weights" in parts and K else None,
        d_texture=rng.standard_normal(npix * K * 3) if "texture" in parts and K else None)


def gpu_backward(renderer, scene, cam, up, err_pixel=None):
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    g = SceneGrads.allocate(scene)
    be = np.zeros(scene.nexels.shape[0]) if err_pixel is not None else None
    renderer.render_backward(ds, cam, fr, up, g, err_pixel, be)
    return (g.prims, g.table, g.w1, g.w2, g.w3, be), fr, ds


def ref_backward(reference, scene, cam, up, err_pixel=None):
    return reference.render_backward(scene, cam, up.d_final, up.d_weights, up.d_texture, err_pixel)


@pytest.mark.parametrize("seed,top_k", [(1, 2), (2, 1), (3, 4), (4, 0), (5, 2)])
def test_random_scene_gradients_match_reference(renderer, reference, seed, top_k):
    scene, cam = reference.random_scene(seed, 60, top_k, 48, 60.0, 3.0)
    up = upstream(cam, top_k, seed)
    err = np.random.default_rng(seed + 100).random(cam.width * cam.height)
    g, _, _ = gpu_backward(renderer, scene, cam, up, err)
    r = ref_backward(reference, scene, cam, up, err)
    rep = compare_grads(g, r)
    print(seed, top_k, {k: f"{v:.1e}" for k, v in rep.items()})
    assert np.abs(r[0]).max() > 0


@pytest.mark.parametrize("parts", [("final",), ("weights",), ("texture",)])
def test_each_upstream_term_alone(renderer, reference, parts):
    scene, cam = reference.random_scene(11, 50, 2, 40, 50.0, 3.0)
    up = upstream(cam, 2, 11, parts)
    g, _, _ = gpu_backward(renderer, scene, cam, up)
    r = ref_backward(reference, scene, cam, up)
    compare_grads(g, r)


@pytest.mark.parametrize("ablation", ["no_gamma", "no_prim_sh", "no_downweight", "min_t0", "alpha_clamp"])
def test_ablations_match_reference(renderer, reference, ablation):
    scene, cam = reference.random_scene(21, 60, 2, 40, 50.0, 3.0, op_lo=0.9 if ablation == "alpha_clamp" else 0.35,
                                        op_hi=0.99999 if ablation == "alpha_clamp" else 0.85)
    st = scene.settings
    if ablation == "no_gamma":
        st.no_gamma = True
    elif ablation == "no_prim_sh":
        st.no_prim_sh = True
    elif ablation == "no_downweight":
        st.no_downweight = True
    elif ablation == "min_t0":
        st.min_transmittance = 0.0
    elif ablation == "alpha_clamp":
        st.alpha_max = 0.9
    up = upstream(cam, 2, 21)
    g, _, _ = gpu_backward(renderer, scene, cam, up)
    r = ref_backward(reference, scene, cam, up)
    compare_grads(g, r)


def test_stump_textured_gradients_match_reference(renderer, reference):
    # grid_init 1e-1: the texture branch carries real gradients
    scene = nx.stump_like(3_000, log2_table=14, grid_init=1e-1)
    cam = nx.ring_camera(3, 256, 96, 64)
    up = upstream(cam, 2, 5)
    err = np.random.default_rng(9).random(cam.width * cam.height)
    g, _, _ = gpu_backward(renderer, scene, cam, up, err)
    r = ref_backward(reference, scene, cam, up, err)
    rep = compare_grads(g, r, GRAD_TOL_TC)
    print({k: f"{v:.1e}" for k, v in rep.items()})


@pytest.mark.parametrize("n,view,size,grid_init,ablation", [
    (10_000, 0, (256, 256), 1e-4, None),          # BASELINE config 1 shape
    (10_000, 17, (160, 120), 1e-1, None),
    (4_000, 40, (128, 96), 1e-1, "no_downweight"),
    (4_000, 90, (128, 96), 1e-1, "no_prim_sh"),
    (4_000, 130, (128, 96), 1e-1, "no_gamma"),
    (4_000, 200, (128, 96), 1e-1, "k4"),
    (4_000, 210, (128, 96), 1e-1, "k3"),           # 128-slot tiles split pixels (3 does not divide 128)
    (4_000, 220, (128, 96), 1e-1, "k1"),
    (6_000, 60, (640, 480), 1e-1, None),          # >= 4 x SMs 16x16 tiles: the 16x16 work-tile kernel
])
def test_stump_field_tc_gradients_match_reference(renderer, reference, n, view, size, grid_init, ablation):
    # the reference field shape (16 levels x 2 x 64 hidden) takes the tcgen05 field backward
    scene = nx.stump_like(n, log2_table=16, grid_init=grid_init)
    st = scene.settings
    if ablation in ("k4", "k3", "k1"):
        st.top_k = int(ablation[1])
    elif ablation:
        setattr(st, ablation, True)
    cam = nx.ring_camera(view, 256, *size)
    up = upstream(cam, st.top_k, view)
    err = np.random.default_rng(view).random(cam.width * cam.height)
    g, _, _ = gpu_backward(renderer, scene, cam, up, err)
    r = ref_backward(reference, scene, cam, up, err)
    rep = compare_grads(g, r, GRAD_TOL_TC)
    print(n, view, ablation, {k: f"{v:.1e}" for k, v in rep.items()})


def test_backward_accumulates_like_the_reference(renderer, reference):
    scene, cam = reference.random_scene(31, 40, 2, 32, 40.0, 3.0)
    up = upstream(cam, 2, 31)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    g = SceneGrads.allocate(scene)
    renderer.render_backward(ds, cam, fr, up, g)
    once = [a.copy() for a in (g.prims, g.table, g.w1, g.w2, g.w3)]
    renderer.render_backward(ds, cam, fr, up, g)
    # every reduction is exact and order-independent: the second pass adds the same
    # bits, so the sum is exactly twice the first
    for a, b in zip((g.prims, g.table, g.w1, g.w2, g.w3), once):
        assert np.array_equal(a, 2 * b)


@pytest.mark.parametrize("case", ["stump_tc", "random_simt", "stump_no_prim_sh"])
def test_backward_is_bit_reproducible(renderer, reference, case):
    """The reference's results are bit-stable for any worker count (threading.hpp:12-16;
    test_train.cpp "training is deterministic run to run"): repeated backward passes of
    the same frame give identical bits, whatever order the GPU's atomics take."""
    if case == "random_simt":
        scene, cam = reference.random_scene(77, 400, 3, 96, 90.0, 3.0)
    else:
        scene = nx.stump_like(30_000, log2_table=16, grid_init=1e-1)
        if case == "stump_no_prim_sh":
            scene.settings.no_prim_sh = True
        cam = nx.ring_camera(23, 256, 320, 240)
    K = scene.settings.top_k
    up = upstream(cam, K, 5)
    err = np.random.default_rng(6).random(cam.width * cam.height)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    runs = []
    for _ in range(3):
        g = SceneGrads.allocate(scene)
        be = np.zeros(scene.nexels.shape[0])
        renderer.render_backward(ds, cam, fr, up, g, err, be)
        runs.append((g.prims, g.table, g.w1, g.w2, g.w3, be))
    assert np.abs(runs[0][0]).max() > 0 and np.abs(runs[0][1]).max() > 0
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            assert np.array_equal(a, b)


_OVERLAP_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import SceneGrads, UpstreamGrads
scene = nx.stump_like(30_000, log2_table=16, grid_init=1e-1)
cam = nx.ring_camera(23, 256, 320, 240)
K, npix = scene.settings.top_k, cam.width * cam.height
rng = np.random.default_rng(5)
up = UpstreamGrads(d_final=rng.standard_normal(npix * 3), d_weights=rng.standard_normal(npix * K),
                   d_texture=rng.standard_normal(npix * K * 3))
r = nx.Renderer(0)
ds = r.upload(scene)
fr = r.frame()
fr.set_backward(True)
r.render(ds, cam, fr)
g = SceneGrads.allocate(scene)
be = np.zeros(scene.nexels.shape[0])
r.render_backward(ds, cam, fr, up, g, np.random.default_rng(6).random(npix), be)
h = hashlib.sha256()
for a in (g.prims, g.table, g.w1, g.w2, g.w3, be):
    h.update(np.ascontiguousarray(a).tobytes())
print(h.hexdigest(), float(np.abs(g.table).max()))
"""


def test_backward_side_stream_is_bit_identical():
    """The table-gradient scatter on the context's side stream (default) and on the
    caller's stream (NX_BWD_OVERLAP=0) give the same bits."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for overlap in ("1", "0"):
        env = dict(os.environ, NX_BWD_OVERLAP=overlap)
        res = subprocess.run([sys.executable, "-c", _OVERLAP_SCRIPT, root], env=env, capture_output=True,
                             text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(res.stdout.strip().splitlines()[-1].split())
    assert float(outs[0][1]) > 0
    assert outs[0][0] == outs[1][0]


def test_backward_of_an_empty_scene_is_zero(renderer, reference):
    """No primitives: the background does not depend on the parameters — every gradient
    (field included) is zero, like the reference's."""
    base = nx.stump_like(2_000, log2_table=16, grid_init=1e-1)
    scene = nx.Scene(np.zeros((0, 60)), base.field, base.settings)
    cam = nx.ring_camera(5, 256, 96, 64)
    up = upstream(cam, scene.settings.top_k, 3)
    g, _, _ = gpu_backward(renderer, scene, cam, up)
    r = ref_backward(reference, scene, cam, up)
    for a in g[:5]:
        assert not np.any(a)
    for a in r[:5]:
        assert not np.any(a)


def test_backward_needs_the_forward_state(renderer, reference):
    scene, cam = reference.random_scene(32, 20, 2, 32, 40.0, 3.0)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    renderer.render(ds, cam, fr)  # backward state not kept
    g = SceneGrads.allocate(scene)
    with pytest.raises(NexelError) as e:
        renderer.render_backward(ds, cam, fr, upstream(cam, 2, 1), g)
    assert e.value.code == "invalid-argument"
    bad = nx.Camera(cam.width, cam.height, -1.0, cam.fy, cam.cx, cam.cy, cam.R, cam.t)
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    with pytest.raises(NexelError) as e:
        renderer.render_backward(ds, bad, fr, upstream(cam, 2, 1), g)
    assert e.value.code == "bad-camera"


def test_value_api_render_backward(reference):
    scene, cam = reference.random_scene(41, 50, 2, 40, 50.0, 3.0)
    res = nx.render(scene, cam)
    up = upstream(cam, 2, 41)
    g = SceneGrads.allocate(scene)
    err = np.random.default_rng(3).random(cam.width * cam.height)
    nx.render_backward(scene, cam, res.fb, up, g, err, res.blended_error)
    r = ref_backward(reference, scene, cam, up, err)
    compare_grads((g.prims, g.table, g.w1, g.w2, g.w3, res.blended_error), r)


def test_backward_reuses_or_rebuilds_the_forward_lists_identically(renderer, reference):
    """render_backward reuses the frame's forward work lists when nothing rebuilt them since
    (same scene version and camera) and re-bins otherwise (renderer.cpp:257): both give the
    same bits."""
    scene = nx.stump_like(20_000, log2_table=14, grid_init=1e-1)
    cam_a, cam_b = nx.ring_camera(3, 256, 256, 192), nx.ring_camera(90, 256, 256, 192)
    K = scene.settings.top_k
    up = upstream(cam_a, K, 9)
    err = np.random.default_rng(4).random(cam_a.width * cam_a.height)
    ds = renderer.upload(scene)
    fa, fb = renderer.frame(), renderer.frame()
    fa.set_backward(True)
    fb.set_backward(True)

    def backward(frame):
        g = SceneGrads.allocate(scene)
        be = np.zeros(scene.nexels.shape[0])
        renderer.render_backward(ds, cam_a, frame, up, g, err, be)
        return (g.prims, g.table, g.w1, g.w2, g.w3, be)

    renderer.render(ds, cam_a, fa)
    reused = backward(fa)               # right after its forward: the lists are reused
    renderer.render(ds, cam_b, fb)      # another frame rebuilds the shared lists
    rebuilt = backward(fa)              # so this one re-bins
    for a, b in zip(reused, rebuilt):
        assert np.array_equal(a, b)
    renderer.render(ds, cam_a, fa)
    again = backward(fa)                # reused again after a fresh forward
    st = scene.settings
    st.no_downweight = True             # a settings change makes a new scene version ...
    ds.set_settings(st)
    st.no_downweight = False
    ds.set_settings(st)
    after_settings = backward(fa)       # ... so this re-bins, with the original settings
    for a, b, c in zip(reused, again, after_settings):
        assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("y0", [472, 904])
def test_config5_scale_band_gradients_match_reference(renderer, reference, y0):
    """BASELINE config 5 scale: the 400K-nexel stump scene with the reference field shape
    (2^20-row hash table, grid_init 1e-1: the texture branch carries real gradients) at
    1920 x 1080, on a 64-row band of the view (a principal-point-shifted camera — every
    pixel keeps its ray, so this is the full frame's backward restricted to those rows;
    the reference's CPU render_backward of the whole frame takes ~30 s). All gradient
    arrays against the reference compiled in place, at the tensor-core tolerance."""
    scene = nx.stump_like(400_000, grid_init=1e-1)
    cam = nx.band_camera(nx.ring_camera(0, 256, 1920, 1080), y0, 64)
    up = upstream(cam, scene.settings.top_k, y0)
    err = np.random.default_rng(y0).random(cam.width * cam.height)
    g, _, _ = gpu_backward(renderer, scene, cam, up, err)
    r = ref_backward(reference, scene, cam, up, err)
    rep = compare_grads(g, r, GRAD_TOL_TC)
    print(y0, {k: f"{v:.1e}" for k, v in rep.items()})
    assert np.count_nonzero(r[0]) > 1000 and np.count_nonzero(r[1]) > 1000


def test_config5_full_frame_backward_is_bit_reproducible(renderer):
    """The whole BASELINE config-5 backward (400K nexels, 1920x1080, reference field
    shape, ~4M buffered slots) twice on the same frame: identical bits (GPU only)."""
    scene = nx.stump_like(400_000, grid_init=1e-1)
    cam = nx.ring_camera(5, 256, 1920, 1080)
    up = upstream(cam, scene.settings.top_k, 5)
    err = np.random.default_rng(5).random(cam.width * cam.height)
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    runs = []
    for _ in range(2):
        g = SceneGrads.allocate(scene)
        be = np.zeros(scene.nexels.shape[0])
        renderer.render_backward(ds, cam, fr, up, g, err, be)
        runs.append((g.prims, g.table, g.w1, g.w2, g.w3, be))
    assert np.abs(runs[0][1]).max() > 0
    for a, b in zip(*runs):
        assert np.array_equal(a, b)
