"""GPU: NX_PRECISION_F64 (the reference's FrameBuffers precision for the colours) against
the reference compiled in place (oracle/_ref), on the same seeded scenes: contributor
decisions bit-exact as always, base / texture / final to 1e-12 — the fp32-colour default
is held to the north star's 1e-3."""
import dataclasses

import numpy as np
import pytest

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import NexelError

pytestmark = pytest.mark.gpu


def _f64(scene):
    s = dataclasses.replace(scene, settings=dataclasses.replace(scene.settings, precision=nx._abi.NX_PRECISION_F64))
    return s


def _render_f64(renderer, scene, cam):
    ds = renderer.upload(scene)
    fr = renderer.frame()
    fr.set_backward(True)
    renderer.render(ds, cam, fr)
    g = fr.download(["ids", "depths", "weights", "texture_f64", "final_f64"])
    base = fr.base_f64()
    fr.close()
    ds.close()
    return g, base


@pytest.mark.parametrize("case", ["config1_textured", "random_k3", "no_prim_sh"])
def test_f64_colours_match_the_reference(renderer, reference, case):
    if case == "config1_textured":
        scene, cam = nx.stump_like(10_000, grid_init=1e-1), nx.ring_camera(0, 256, 256, 256)
    elif case == "random_k3":
        scene, cam = nx.stump_like(6_000, grid_init=1e-1, seed=11), nx.ring_camera(37, 256, 160, 120)
        scene.settings.top_k = 3
    else:
        scene, cam = nx.stump_like(6_000, grid_init=1e-1, seed=5), nx.ring_camera(90, 256, 160, 120)
        scene.settings.no_prim_sh = True
    g, base = _render_f64(renderer, _f64(scene), cam)
    r = reference.render(scene, cam)
    assert np.array_equal(g.ids, r.ids)
    for name, a, b in (("base", base, r.base), ("texture", g.texture_f64, r.texture), ("final", g.final_f64,
                                                                                        r.final_img)):
        err = float(np.abs(a - b).max())
        print(case, name, err)
        assert err <= 1e-12, (name, err)
    assert float(np.abs(g.weights - r.weights).max()) <= 1e-13


def test_f64_scenes_are_render_only(renderer):
    scene = _f64(nx.stump_like(2_000, log2_table=12))
    ds = renderer.upload(scene)
    with pytest.raises(NexelError):
        renderer.optimizer(ds)
    ds.close()
