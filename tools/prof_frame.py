"""Profiling driver: renders config-2 views (400K nexels, 1920x1080, K=2) a few times.

Used under ncu on the GPU box, e.g.
  ncu --set full --clock-control none --import-source on -k regex:texture_kernel -s 2 -c 1 \
      -o gpurun_out/prof_texture python tools/prof_frame.py
Numbers printed under a profiler are never bench values.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2512_13796_b200 as nx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frames", type=int, default=4)
p.add_argument("--nexels", type=int, default=400_000)
p.add_argument("--width", type=int, default=1920)
p.add_argument("--height", type=int, default=1080)
p.add_argument("--grid-init", type=float, default=1e-4)
a = p.parse_args()

scene = nx.stump_like(a.nexels, grid_init=a.grid_init)
r = nx.Renderer(0)
ds = r.upload(scene)
fr = r.frame()
for i in range(a.frames):
    r.render(ds, nx.ring_camera(i, 256, a.width, a.height), fr)
r.synchronize()
print(fr.stats())
