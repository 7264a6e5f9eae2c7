"""GPU: NEXL checkpoints (checkpoint.cpp:99-271) written by the reference's own
save_checkpoint load straight into a device scene (nx_scene_load_nexl) and render
exactly like the in-memory scene they came from; the reference's error codes
(missing-file, bad-checkpoint) for absent, truncated and foreign files. Mirrors the
reference's round-trip test (proj/tests/test_io.cpp:297-302)."""
import numpy as np
import pytest

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import NexelError
from parity import compare_frames

pytestmark = pytest.mark.gpu


def test_reference_checkpoint_renders_bit_identically(renderer, reference, tmp_path):
    scene = nx.stump_like(5_000, log2_table=14, grid_init=1e-1)  # every value fp32-exact
    scene.settings.top_k = 3
    scene.settings.min_transmittance = 2e-4
    cams = [nx.ring_camera(i * 40, 256, 160, 96) for i in range(4)]
    path = tmp_path / "scene.nexl"
    reference.save_checkpoint(scene, str(path), cams, iteration=1234)
    ds, meta, loaded_cams = renderer.load_checkpoint(str(path))
    assert meta["iteration"] == 1234 and meta["n_nexels"] == 5_000 and not meta["has_optimizer"]
    assert meta["settings"].top_k == 3 and meta["settings"].min_transmittance == 2e-4
    assert meta["extent"] == scene.extent and meta["n_hidden"] == 64
    assert [c.name for c in loaded_cams] == ["cam0", "cam1", "cam2", "cam3"]
    for c, lc in zip(cams, loaded_cams):
        assert np.array_equal(lc.to_c().R[:], c.to_c().R[:]) and lc.width == c.width
    mem = renderer.upload(scene)
    fa, fb = renderer.frame(), renderer.frame()
    for cam in loaded_cams[1:3]:
        renderer.render(ds, cam, fa)
        renderer.render(mem, cam, fb)
        a, b = fa.download(), fb.download()
        for k in ("ids", "depths", "weights", "base", "texture", "final_img", "residual"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), k
        compare_frames(a, reference.render(scene, cam))


def test_checkpoint_error_codes(renderer, reference, tmp_path):
    with pytest.raises(NexelError) as e:
        renderer.load_checkpoint(str(tmp_path / "absent.nexl"))
    assert e.value.code == "missing-file"
    scene = nx.stump_like(500, log2_table=10)
    path = tmp_path / "ok.nexl"
    reference.save_checkpoint(scene, str(path), [nx.ring_camera(0, 256, 32, 32)])
    data = path.read_bytes()
    (tmp_path / "cut.nexl").write_bytes(data[: len(data) // 2])
    with pytest.raises(NexelError) as e:
        renderer.load_checkpoint(str(tmp_path / "cut.nexl"))
    assert e.value.code == "bad-checkpoint" and "truncated" in str(e.value)
    (tmp_path / "foreign.nexl").write_bytes(b"PNG!" + data[4:])
    with pytest.raises(NexelError) as e:
        renderer.load_checkpoint(str(tmp_path / "foreign.nexl"))
    assert e.value.code == "bad-checkpoint" and "magic" in str(e.value)
    bad = bytearray(data)
    bad[4] = 7  # version
    (tmp_path / "v7.nexl").write_bytes(bytes(bad))
    with pytest.raises(NexelError) as e:
        renderer.load_checkpoint(str(tmp_path / "v7.nexl"))
    assert e.value.code == "bad-checkpoint" and "version" in str(e.value)
