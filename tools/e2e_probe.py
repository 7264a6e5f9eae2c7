"""Where does the e2e step time go? render-only, download-only, and the pipelined
render+download loop with 2 and 3 frames in flight (config 2)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi

scene = nx.stump_like(400_000)
r = nx.Renderer(0)
ds = r.upload(scene)
W, H, K = 1920, 1080, 2
cams = [nx.ring_camera(v, 256, W, H) for v in range(32)]
npix = W * H
host = {
    "base": torch.empty(npix * 3, dtype=torch.float32, pin_memory=True),
    "ids": torch.empty(npix * K, dtype=torch.int32, pin_memory=True),
    "depths": torch.empty(npix * K, dtype=torch.float64, pin_memory=True),
    "weights": torch.empty(npix * K, dtype=torch.float64, pin_memory=True),
    "texture": torch.empty(npix * K * 3, dtype=torch.float32, pin_memory=True),
    "final_img": torch.empty(npix * 3, dtype=torch.float32, pin_memory=True),
    "residual": torch.empty(npix, dtype=torch.float32, pin_memory=True),
}
hf = _abi.nx_host_frame()
for k, t in host.items():
    setattr(hf, k, t.data_ptr())
stream = torch.cuda.ExternalStream(r.stream)


def timed(fn, n=20):
    for i in range(3):
        fn(i)
    r._check(r.lib.nx_ctx_join(r.ctx))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(n):
        fn(i)
    r._check(r.lib.nx_ctx_join(r.ctx))
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (time.perf_counter() - t0) * 1e3 / n


for nf in (2, 3, 4):
    frames = [r.frame() for _ in range(nf)]
    print(f"frames={nf} render only      {timed(lambda i: r.render(ds, cams[i % 32], frames[i % nf]))}")
    def both(i):
        f = frames[i % nf]
        r.render(ds, cams[i % 32], f)
        r._check(r.lib.nx_frame_download(r.ctx, f.handle, C.byref(hf), None))
    print(f"frames={nf} render+download  {timed(both)}")
    print(f"frames={nf} download only    {timed(lambda i: r._check(r.lib.nx_frame_download(r.ctx, frames[i % nf].handle, C.byref(hf), None)))}")
    for f in frames:
        f.close()

# download duration when overlapped with rendering: events on the copy stream
frames = [r.frame() for _ in range(2)]
for i in range(4):
    r.render(ds, cams[i], frames[i % 2])
r._check(r.lib.nx_ctx_join(r.ctx))
torch.cuda.synchronize()
cs = torch.cuda.Stream()
evs = []
t_start = torch.cuda.Event(enable_timing=True)
t_start.record(stream)
for i in range(12):
    f = frames[i % 2]
    r.render(ds, cams[i % 32], f)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # explicit copy stream: wait for the frame, time the copies
    r._check(r.lib.nx_ctx_join(r.ctx))
    ev_ready = torch.cuda.Event()
    ev_ready.record(stream)
    cs.wait_event(ev_ready)
    a.record(cs)
    r._check(r.lib.nx_frame_download(r.ctx, f.handle, C.byref(hf), C.c_void_p(cs.cuda_stream)))
    b.record(cs)
    evs.append((a, b))
torch.cuda.synchronize()
print("download ms when overlapped:", [round(a.elapsed_time(b), 2) for a, b in evs])
print("gaps between downloads:", [round(evs[i][1].elapsed_time(evs[i + 1][0]), 2) for i in range(len(evs) - 1)])
