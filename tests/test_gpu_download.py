"""GPU: the fp32 weights download (nx_host_frame.weights_f32). Display frames composite in
fp32 (the certified march), so their slot weights are fp32 values: narrowing them on the
device halves their PCIe bytes without losing a bit, except at the pixels the exact redo
re-rendered (fp64 weights, rounded). Checked against the fp64 download of the same frame."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi

pytestmark = pytest.mark.gpu

W, H = 640, 480


@pytest.fixture(scope="module")
def rendered():
    r = nx.Renderer(0)
    ds = r.upload(nx.stump_like(40_000, grid_init=1e-1))
    f = r.frame()
    r.render(ds, nx.ring_camera(17, 256, W, H), f)
    yield r, f
    f.close()
    ds.close()
    r.close()


def _download(r, f, **bufs):
    hf = _abi.nx_host_frame()
    for k, v in bufs.items():
        setattr(hf, k, v)
    st = r.lib.nx_frame_download(r.ctx, f.handle, C.byref(hf), None)
    if st == _abi.NX_OK:
        r._check(r.lib.nx_ctx_synchronize(r.ctx))
    return st


def test_fp32_weights_are_the_fp64_weights_narrowed(rendered):
    r, f = rendered
    g = f.download()
    K = f.view().top_k
    w32 = torch.zeros(W * H * K, dtype=torch.float32, pin_memory=True)
    assert _download(r, f, weights_f32=w32.data_ptr()) == _abi.NX_OK
    w32 = w32.numpy()
    assert np.array_equal(w32, g.weights.astype(np.float32))
    # lossless except the exactly redone pixels (fp64 weights from the exact composite)
    lost = np.count_nonzero(w32.astype(np.float64) != g.weights)
    redo = f.stats()["redo_tiles"]
    print(f"slots {w32.size}, occupied {np.count_nonzero(g.ids >= 0)}, rounded {lost}, redo pixels {redo}")
    assert lost <= K * redo
    assert np.count_nonzero(g.ids >= 0) > W * H // 2


def test_fp32_weights_need_pinned_memory_and_exclude_fp64(rendered):
    r, f = rendered
    K = f.view().top_k
    pageable = np.zeros(W * H * K, np.float32)
    assert _download(r, f, weights_f32=pageable.ctypes.data) == _abi.NX_INVALID_ARGUMENT
    w32 = torch.zeros(W * H * K, dtype=torch.float32, pin_memory=True)
    w64 = np.zeros(W * H * K)
    st = _download(r, f, weights_f32=w32.data_ptr(), weights=w64.ctypes.data)
    assert st == _abi.NX_INVALID_ARGUMENT
