"""CPU: the plain-C oracle (oracle/nexel_oracle.c) pinned against golden fixtures
produced by the reference itself (tests/golden/make_golden.py runs the reference
compiled in place). Bit-exact discrete outputs, fp64 values to ~1e-12."""
import glob
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import load  # noqa: E402

import paper_2512_13796_b200 as nx  # noqa: E402

CASES = sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(HERE, "golden", "*.npz")))
INPUT_CASES = [c for c in CASES if c != "config1"]


def test_fixture_inventory():
    assert "config1" in CASES and "stump_2k" in CASES and len(INPUT_CASES) >= 14


@pytest.mark.parametrize("case", INPUT_CASES)
def test_oracle_matches_reference_golden(oracle, case):
    z, scene, cam, _ = load(case)
    fb = oracle.render(scene, cam)
    assert np.array_equal(fb.ids, z["ids"]), "slot ids"
    np.testing.assert_allclose(fb.depths, z["depths"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(fb.weights, z["weights"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(fb.residual, z["residual"], rtol=1e-12, atol=1e-15)
    for k in ("base", "texture", "final_img"):
        np.testing.assert_allclose(getattr(fb, k), z[k], rtol=0, atol=1e-12, err_msg=k)
    if "naive" in z:  # thin scenes: the brute-force oracle agrees (acceptance.cpp:92-130)
        assert np.abs(fb.final_img - z["naive"]).max() <= 1e-6


def test_oracle_tile_lists_match_reference_golden(oracle):
    z, scene, cam, _ = load("stump_2k")
    off, ids, _, _ = oracle.tile_lists(scene, cam)
    assert np.array_equal(off, z["tile_offsets"])
    assert np.array_equal(ids, z["tile_ids"])


def test_config1_oracle_matches_reference_golden(oracle):
    """BASELINE config 1 (10K nexels, 256x256): P = 143,383, ids and
    tile lists bit-exact, final image as stored (fp32) by the reference run."""
    z, _, cam, _ = load("config1")
    scene = nx.stump_like(10_000)
    off, ids, _, _ = oracle.tile_lists(scene, cam)
    assert off[-1] == 143_383
    assert np.array_equal(off, z["tile_offsets"]) and np.array_equal(ids, z["tile_ids"])
    fb = oracle.render(scene, cam)
    assert fb.stats["n_straddlers"] == 468
    assert np.array_equal(fb.ids, z["ids"])
    np.testing.assert_allclose(fb.weights, z["weights"], rtol=1e-12, atol=1e-15)
    assert np.abs(fb.final_img - z["final_img"]).max() < 1e-6
    assert abs(fb.final_img.sum() - float(z["final_sum"][0])) < 1e-6
    assert abs(fb.final_img.sum() - 92174.708823425) < 1e-3  # SURVEY.md Appendix A self-check


def test_oracle_errors_follow_the_reference(oracle):
    from oracle.pyoracle import OracleError
    _, scene, cam, _ = load("random_k2")
    bad = nx.Scene(scene.nexels, scene.field, nx.RenderSettings(top_k=9))
    with pytest.raises(OracleError) as e:
        oracle.render(bad, cam)
    assert e.value.code == "bad-settings"
    nex = scene.nexels.copy()
    nex[3, 5] = np.inf
    with pytest.raises(OracleError) as e:
        oracle.render(nx.Scene(nex, scene.field, scene.settings), cam)
    assert e.value.code == "bad-primitive" and "primitive 3" in str(e.value)
    c2 = nx.Camera(cam.width, cam.height, -1.0, cam.fy, cam.cx, cam.cy, cam.R, cam.t)
    with pytest.raises(OracleError) as e:
        oracle.render(scene, c2)
    assert e.value.code == "bad-camera"


def test_oracle_topk_rules(oracle):
    """test_renderer.cpp:15-52 known answers."""
    import ctypes as C
    L = oracle.lib

    def run(k, ws):
        n = len(ws)
        ids = np.arange(n, dtype=np.int32)
        w = np.asarray(ws, np.float64)
        t = 1.0 + np.arange(n, dtype=np.float64)
        oi = np.full(8, -2, np.int32)
        ow = np.zeros(8)
        size = L.orc_topk(k, n, ids.ctypes.data_as(C.POINTER(C.c_int32)), w.ctypes.data_as(C.POINTER(C.c_double)),
                          t.ctypes.data_as(C.POINTER(C.c_double)), oi.ctypes.data_as(C.POINTER(C.c_int32)),
                          ow.ctypes.data_as(C.POINTER(C.c_double)))
        return size, oi[:k], ow[:k]

    size, ids, w = run(2, [0.5, 0.7, 0.6])
    assert size == 2 and list(ids) == [1, 2] and w[0] == 0.7
    assert list(run(2, [0.5, 0.5, 0.5])[1]) == [0, 1]
    assert list(run(1, [0.5, 0.5])[1]) == [0]
    size, ids, _ = run(2, [0.4])
    assert size == 1 and ids[1] == -1
    rng = np.random.default_rng(71)
    for _ in range(2000):  # tie-heavy sequences == stable full sort (test_renderer.cpp:54-78)
        n = int(rng.integers(1, 13))
        k = int(rng.integers(1, 9))
        ws = rng.choice([0.1, 0.2, 0.3, 0.4], n)
        size, ids, _ = run(k, ws)
        want = sorted(range(n), key=lambda i: -ws[i])[:k]
        assert size == min(k, n) and list(ids[:size]) == want


def test_oracle_kernel_known_answers(oracle):
    """test_geometry.cpp:112-199, test_field.cpp:17-42 known answers."""
    L = oracle.lib
    rng = np.random.default_rng(5)
    import math
    for _ in range(100):  # gamma = 1 is bit-identical to the Gaussian (libm exp, as the reference)
        u, v, o = float(rng.uniform(-3, 3)), float(rng.uniform(-3, 3)), float(rng.uniform(0.01, 1))
        assert L.orc_eval_kernel(u, v, o, 1.0, 1.0) == o * math.exp(-0.5 * (u * u + v * v))
    for o, g in ((0.7, 1.0), (0.3, 2.5), (0.99, 4.0)):
        r = L.orc_support_radius(o, g)
        assert abs(L.orc_eval_kernel(r, 0.0, o, g, g) - 1 / 255) < 1e-12
    assert [L.orc_map_positive(x) for x in (0, 1, -1, 2, -2)] == [0, 1, 2, 3, 4]
    a, b, c = 3, -7, 11
    want = (3 * 2 - 1) ^ ((14 * 2654435761) & 0xFFFFFFFF) ^ (((11 * 2 - 1) * 805459861) & 0xFFFFFFFF)
    assert L.orc_hash_cell(a, b, c, 1 << 20) == want & ((1 << 20) - 1)
