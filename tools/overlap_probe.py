"""Does a concurrent D2H copy slow the render (or vice versa)?"""
import sys
import torch
sys.path.insert(0, '.')
import paper_2512_13796_b200 as nx

scene = nx.stump_like(400_000)
r = nx.Renderer(0)
ds = r.upload(scene)
cams = [nx.ring_camera(v, 256, 1920, 1080) for v in range(32)]
frames = [r.frame() for _ in range(2)]
stream = torch.cuda.ExternalStream(r.stream)
src = torch.empty(191 * 1024 * 1024, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src, device="cpu").pin_memory()
cs = torch.cuda.Stream()
for i in range(4):
    r.render(ds, cams[i], frames[i % 2])
r.synchronize()
for mode in ("render", "copy", "both"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    c0.record(cs)
    for i in range(10):
        if mode in ("copy", "both"):
            with torch.cuda.stream(cs):
                dst.copy_(src, non_blocking=True)
        if mode in ("render", "both"):
            r.render(ds, cams[i % 32], frames[i % 2])
    r._check(r.lib.nx_ctx_join(r.ctx))
    e1.record(stream)
    c1.record(cs)
    torch.cuda.synchronize()
    print(mode, "render stream ms/iter", round(e0.elapsed_time(e1) / 10, 3), "copy stream ms/iter", round(c0.elapsed_time(c1) / 10, 3))
