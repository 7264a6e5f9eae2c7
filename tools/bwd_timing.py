"""Times render + render_backward at config 2 (device-resident, CUDA events)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import SceneGrads, UpstreamGrads, _abi
import ctypes as C

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
W, H = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1920, 1080)
scene = nx.stump_like(n, grid_init=1e-1)
cam = nx.ring_camera(0, 256, W, H)
r = nx.Renderer(0)
ds = r.upload(scene)
fr = r.frame()
fr.set_backward(True)
K = scene.settings.top_k
npix = W * H
dev = torch.device('cuda')
g = torch.Generator(device=dev).manual_seed(0)
d_final = torch.randn(npix * 3, dtype=torch.float64, device=dev, generator=g)
d_weights = torch.randn(npix * K, dtype=torch.float64, device=dev, generator=g)
d_texture = torch.randn(npix * K * 3, dtype=torch.float64, device=dev, generator=g)
err = torch.rand(npix, dtype=torch.float64, device=dev, generator=g)
f = scene.field
gp = torch.zeros(n * 60, dtype=torch.float64, device=dev)
gt = torch.zeros(f.grid.param_count(), dtype=torch.float64, device=dev)
g1 = torch.zeros(np.size(f.w1), dtype=torch.float64, device=dev)
g2 = torch.zeros(np.size(f.w2), dtype=torch.float64, device=dev)
g3 = torch.zeros(np.size(f.w3), dtype=torch.float64, device=dev)
be = torch.zeros(n, dtype=torch.float64, device=dev)
u = _abi.nx_upstream(d_final.data_ptr(), d_weights.data_ptr(), d_texture.data_ptr())
gg = _abi.nx_grads(gp.data_ptr(), gt.data_ptr(), g1.data_ptr(), g2.data_ptr(), g3.data_ptr())
c = cam.to_c()
lib = r.lib
stream = r.stream
ts = torch.cuda.ExternalStream(stream)


def step(bwd=True):
    r._check(lib.nx_render(r.ctx, ds.handle, C.byref(c), fr.handle, C.c_void_p(stream)))
    if bwd:
        r._check(lib.nx_render_backward(r.ctx, ds.handle, C.byref(c), fr.handle, C.byref(u), C.byref(gg),
                                        C.c_void_p(err.data_ptr()), C.c_void_p(be.data_ptr()), C.c_void_p(stream)))


for bwd in (False, True):
    for _ in range(2):
        step(bwd)
    r.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record(ts)
    for _ in range(steps):
        step(bwd)
    e1.record(ts)
    r.synchronize()
    torch.cuda.synchronize()
    print(f"{'fwd+bwd' if bwd else 'fwd'}: {e0.elapsed_time(e1) / steps:.3f} ms/step", flush=True)
print("grad norms", float(gp.abs().max()), float(gt.abs().max()), float(g1.abs().max()))
