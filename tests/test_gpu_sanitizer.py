"""GPU: compute-sanitizer memcheck and racecheck over a config-1-sized render (the
forward: preprocess, sorts, composite, texture) and a render_backward, run in a
subprocess; both must report 0 errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2512_13796_b200 as nx
scene = nx.stump_like(10_000, log2_table=16, grid_init=1e-1)
cam = nx.ring_camera(0, 256, 256, 256)
r = nx.Renderer(0)
ds = r.upload(scene)
fr = r.frame()
fr.set_backward(True)
r.render(ds, cam, fr)
g = fr.download()
if sys.argv[2] == "backward":
    npix = 256 * 256
    rng = np.random.default_rng(1)
    up = nx.UpstreamGrads(rng.uniform(-1, 1, npix * 3), rng.uniform(-1, 1, npix * 2), rng.uniform(-1, 1, npix * 6))
    grads = nx.SceneGrads.allocate(scene)
    r.render_backward(ds, cam, fr, up, grads)
    assert np.isfinite(grads.prims).all()
print("ok", int((g.ids >= 0).sum()))
"""


@pytest.mark.slow
@pytest.mark.parametrize("tool,what", [("memcheck", "forward"), ("memcheck", "backward"), ("racecheck", "forward")])
def test_compute_sanitizer_clean(tmp_path, tool, what):
    script = tmp_path / "run.py"
    script.write_text(_SCRIPT)
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "99", sys.executable, str(script), ROOT, what]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    tail = (p.stdout + p.stderr)[-3000:]
    if p.returncode != 0 and "closed on this pool" in tail:
        # the GPU pool's compute-sanitizer wrapper refuses every run (it has left GPUs
        # needing a reset); the bounds are covered by the parity tests' exact lists
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + tail.strip()[:160])
    assert p.returncode == 0, tail
    out = p.stdout + p.stderr
    assert "ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out, tail
