"""Frame time with the default two-stream pipelining vs one stream (no overlap of a
frame's texture pass with the next frame's collection). Config 2. NX_PROBE_FRAMES sets
the number of frames in flight (default 2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_13796_b200 as nx  # noqa: E402

NF = int(os.environ.get("NX_PROBE_FRAMES", "2"))
scene = nx.stump_like(400_000)
r = nx.Renderer(0)
ds = r.upload(scene)
frames = [r.frame() for _ in range(NF)]
cams = [nx.ring_camera(i, 256, 1920, 1080) for i in range(256)]
for mode in ("two-stream", "one-stream", "two-stream", "one-stream"):
    st = r.stream if mode == "one-stream" else 0
    for i in range(5):
        r.render(ds, cams[i], frames[i % NF], st)
    r.synchronize()
    t0 = time.perf_counter()
    n = 60
    for i in range(n):
        r.render(ds, cams[i], frames[i % NF], st)
    r.synchronize()
    print(mode, round((time.perf_counter() - t0) / n * 1e3, 3), "ms/frame")
