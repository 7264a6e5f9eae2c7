"""Dumps render_backward gradients for a stump scene with the upstream gradient on
a few slots only (debugging the field backward paths)."""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import SceneGrads, UpstreamGrads

out = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "one"
scene = nx.stump_like(4000, log2_table=16, grid_init=1e-1)
cam = nx.ring_camera(40, 256, 128, 96)
r = nx.Renderer(0)
ds = r.upload(scene)
fr = r.frame()
fr.set_backward(True)
r.render(ds, cam, fr)
fb = fr.download()
K = 2
npix = cam.width * cam.height
dt = np.zeros(npix * K * 3)
occ = np.nonzero(fb.ids >= 0)[0]
rng = np.random.default_rng(0)
if mode == "one":
    sel = occ[[len(occ) // 2]]
elif mode == "row":
    sel = occ[len(occ) // 2: len(occ) // 2 + 128]
elif mode == "same_cta":   # two tiles processed by the same CTA, one after the other
    t0 = 10
    sel = [s for s in occ if s // 128 in (t0, t0 + 148)]
elif mode == "adjacent":   # two tiles of different CTAs
    t0 = (len(occ) // 2) // 128
    sel = [s for s in occ if s // 128 in (t0, t0 + 1)]
elif mode == "first148":  # one tile per CTA
    sel = [s for s in occ if s // 128 < 148]
elif mode == "second":  # the CTAs' second tiles only
    sel = [s for s in occ if s // 128 >= 148]
else:
    sel = occ
for s in sel:
    dt[s * 3: s * 3 + 3] = rng.standard_normal(3)
g = SceneGrads.allocate(scene)
r.render_backward(ds, cam, fr, UpstreamGrads(d_texture=dt), g)
np.savez(out, prims=g.prims, table=g.table, w1=g.w1, w2=g.w2, w3=g.w3, sel=sel)
