"""Kernel timeline of a few config-2 frames (CUPTI via torch.profiler): per kernel start,
duration and stream, the GPU-busy fraction and the idle gaps. Usage:
python tools/timeline.py [--one-stream] [--frames N] [--out gpurun_out/timeline.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2512_13796_b200 as nx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--one-stream", action="store_true")
p.add_argument("--frames", type=int, default=6)
p.add_argument("--out", default="gpurun_out/timeline.json")
p.add_argument("--download", action="store_true")
a = p.parse_args()

scene = nx.stump_like(400_000)
r = nx.Renderer(0)
ds = r.upload(scene)
frames = [r.frame(), r.frame()]
cams = [nx.ring_camera(i, 256, 1920, 1080) for i in range(256)]
st = r.stream if a.one_stream else 0
for i in range(6):
    r.render(ds, cams[i], frames[i % 2], st)
r.synchronize()
torch.cuda.init()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(a.frames):
        r.render(ds, cams[10 + i], frames[i % 2], st)
    r.synchronize()
prof.export_chrome_trace(a.out)
ev = [e for e in json.load(open(a.out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
t_end = max(e["ts"] + e["dur"] for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for e in ev:
    s, d = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, d
    else:
        cur_e = max(cur_e, d)
busy += cur_e - cur_s
span = t_end - t0
print(f"frames {a.frames}  span {span / 1e3:.3f} ms  per frame {span / a.frames / 1e3:.3f} ms  "
      f"busy {busy / span * 100:.1f}%  kernels {len(ev)}")
agg = {}
for e in ev:
    n = e["name"].split("(")[0].replace("void ", "").split("<")[0][-40:]
    x = agg.setdefault(n, [0, 0.0])
    x[0] += 1
    x[1] += e["dur"]
for n, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:42s} {c / a.frames:5.1f}/frame {d / a.frames:8.1f} us/frame")
gaps = []
prev_end = None
for e in ev:
    if prev_end is not None and e["ts"] > prev_end + 2:
        gaps.append((e["ts"] - prev_end, e["name"].split("(")[0][-40:]))
    prev_end = e["ts"] + e["dur"] if prev_end is None else max(prev_end, e["ts"] + e["dur"])
gaps.sort(reverse=True)
print("largest idle gaps (us, next kernel):", [(round(g, 1), n) for g, n in gaps[:12]])
print("total idle", round(sum(g for g, _ in gaps) / a.frames, 1), "us/frame")
