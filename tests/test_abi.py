"""CPU: the C-ABI library loads, exports every symbol include/nexel_b200.h declares,
and its host-side logic (synthetic inputs, status names, no-device behaviour)
works without a GPU. No kernel is launched here."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "nexel_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    syms = header_symbols()
    assert len(syms) >= 29
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _abi.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_status_names_match_reference_error_codes():
    lib = _abi.load()
    assert lib.nx_status_name(_abi.NX_BAD_SETTINGS) == b"bad-settings"
    assert lib.nx_status_name(_abi.NX_BAD_CAMERA) == b"bad-camera"
    assert lib.nx_status_name(_abi.NX_BAD_PRIMITIVE) == b"bad-primitive"
    assert lib.nx_version().startswith(b"nexel-b200")


def test_settings_defaults_match_reference():
    lib = _abi.load()
    s = _abi.nx_settings()
    lib.nx_settings_default(C.byref(s))
    r = nx.RenderSettings()
    assert (s.top_k, s.tile, s.near_eps, s.alpha_max, s.min_transmittance) == \
           (r.top_k, r.tile, r.near_eps, r.alpha_max, r.min_transmittance) == (2, 16, 1e-3, 0.999, 1e-4)


def test_no_device_is_reported_not_faked():
    lib = _abi.load()
    n = C.c_int(-1)
    lib.nx_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is visible")
    ctx = C.c_void_p()
    assert lib.nx_ctx_create(0, C.byref(ctx)) == _abi.NX_NO_DEVICE
    with pytest.raises(nx.NexelError) as e:
        nx.Renderer(0)
    assert e.value.code == "no-device"


def test_stump_like_is_deterministic_and_f32_exact():
    a = nx.stump_like(3_000, log2_table=10)
    b = nx.stump_like(3_000, log2_table=10)
    assert np.array_equal(a.nexels, b.nexels) and np.array_equal(a.field.table, b.field.table)
    for arr in (a.nexels, a.field.table, a.field.w1, a.field.w2, a.field.w3):
        assert np.array_equal(arr, arr.astype(np.float32).astype(np.float64))
    # 55% ground (z = 0), 15% cylinder, 30% dome
    assert np.count_nonzero(a.nexels[:, 2] == 0.0) == int(0.55 * 3000)
    g = a.field.grid
    assert (g.levels, g.log2_table, g.features, a.field.n_hidden) == (16, 10, 2, 64)
    assert g.base_scale == 1.0 / 16.0 and abs(g.growth ** 15 - 32768.0) < 1e-9
    c = nx.stump_like(3_000, log2_table=10, seed=99)
    assert not np.array_equal(a.nexels, c.nexels)


def test_stump_like_field_matches_reference_init(reference):
    """TextureField::init / HashGridConfig::for_extent of the reference produce the
    same table and MLP weights (up to the fp32 rounding the synth applies)."""
    ours = nx.stump_like(100, log2_table=8, grid_init=1e-4).field
    theirs = reference.field_for_extent(2513, 16.0, 16, 8, 1e-4)
    assert theirs.grid.base_scale == ours.grid.base_scale and theirs.grid.growth == ours.grid.growth
    for k in ("table", "w1", "w2", "w3"):
        t = getattr(theirs, k).astype(np.float32).astype(np.float64)
        assert np.array_equal(t, getattr(ours, k)), k


def test_ring_camera_is_a_valid_look_at():
    for i in (0, 17, 255):
        cam = nx.ring_camera(i, 256, 1920, 1080)
        R = np.asarray(cam.R)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12) and np.linalg.det(R) > 0
        th = 2 * math.pi * i / 256 + 0.37
        eye = np.array([3 * math.cos(th), 3 * math.sin(th), 1.2 + 0.2 * math.sin(3 * th)])
        assert np.allclose(cam.position(), eye, atol=1e-12)
        assert (cam.fx, cam.cx, cam.cy) == (0.8 * 1920, 960.0, 540.0)
        fwd = np.array([0, 0, 0.4]) - eye
        assert np.allclose(R[2], fwd / np.linalg.norm(fwd), atol=1e-12)


def test_hash_grid_config_for_extent():
    g = nx.HashGridConfig.for_extent(2.0)
    assert g.base_scale == 0.5 and abs(g.base_scale * g.growth ** 15 - 16384.0) < 1e-6
    assert g.param_count() == 16 * (1 << 20) * 2


def test_nexl_header_reader_on_a_reference_checkpoint(tmp_path):
    # host-side half of nx_scene_load_nexl: cameras and error codes, no GPU needed
    from oracle.pyoracle import Reference
    try:
        ref = Reference()
    except ImportError as e:
        pytest.skip(str(e))
    lib = _abi.load()
    scene = nx.stump_like(300, log2_table=8)
    cams = [nx.ring_camera(i, 256, 40 + i, 30) for i in range(3)]
    path = str(tmp_path / "s.nexl")
    ref.save_checkpoint(scene, path, cams, iteration=7)
    n = C.c_int(0)
    out = (_abi.nx_camera * 3)()
    names = (C.c_char * 64 * 3)()
    assert lib.nx_nexl_cameras(path.encode(), out, names, 3, C.byref(n)) == _abi.NX_OK
    assert n.value == 3
    for i in range(3):
        assert bytes(names[i]).split(b"\0")[0] == f"cam{i}".encode()
        assert out[i].width == 40 + i and list(out[i].R) == list(cams[i].to_c().R)
    assert lib.nx_nexl_cameras(str(tmp_path / "none.nexl").encode(), None, None, 0, C.byref(n)) == \
        _abi.NX_MISSING_FILE
    assert lib.nx_status_name(_abi.NX_BAD_CHECKPOINT) == b"bad-checkpoint"
