import sys
import numpy as np
a = np.load(sys.argv[1]); b = np.load(sys.argv[2])
for k in ("w3", "w2", "w1", "table", "prims"):
    x, y = a[k], b[k]
    s = np.abs(y).max()
    e = np.abs(x - y)
    print(k, "scale", s, "max err", e.max(), "rel", e.max() / max(s, 1e-300))
    if k in ("w2", "w1", "w3"):
        sh = (48, 64) if k == "w3" else ((64, 64) if k == "w2" else (64, 32))
        E = (e / max(s, 1e-300)).reshape(sh)
        print("  worst rows", np.argsort(-E.max(1))[:8], "worst cols", np.argsort(-E.max(0))[:8])
        print("  ratio sample", (x.reshape(sh)[:2, :6] / np.where(y == 0, 1, y).reshape(sh)[:2, :6]))
