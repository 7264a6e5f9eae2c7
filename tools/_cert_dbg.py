import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from test_gpu_fastmath import _run
rng = np.random.default_rng(21)
n = 3_000_000
g = np.where(rng.random(n) < 0.1, 1.0, 1.0 + rng.uniform(0, 5, n))
gy = np.where(rng.random(n) < 0.1, 1.0, 1.0 + rng.uniform(0, 5, n))
o = np.exp(rng.uniform(np.log(0.004), np.log(0.999), n))
ru = (2 * np.log(np.maximum(o * 255, 1.0001))) ** (1 / (2 * g))
u = rng.uniform(-1.05, 1.05, n) * ru * np.where(rng.random(n) < 0.02, 1e-6, 1.0)
v = rng.uniform(-1.05, 1.05, n) * (2 * np.log(np.maximum(o * 255, 1.0001))) ** (1 / (2 * gy))
u[:1000] = 0.0
x = np.stack([u, v, g, gy, o], 1).reshape(-1)
y = _run(4, x).reshape(-1, 5)
a32, eps, oma32, eps_oma, a64 = y.T
r = np.abs(a32 - a64) / (eps * np.maximum(a64, 1e-30))
bad = np.argsort(-r)[:10]
for i in bad:
    print(f"ratio {r[i]:.3f} u {u[i]:.3e} v {v[i]:.3e} g {g[i]:.3f} gy {gy[i]:.3f} o {o[i]:.4f} a32 {a32[i]:.6e} a64 {a64[i]:.6e} eps {eps[i]:.2e}")
oma64 = 1 - a64
ok = oma64 > 1e-6
r2 = np.abs(oma32 - oma64) / (eps_oma * oma64)
r2[~ok] = 0
for i in np.argsort(-r2)[:5]:
    print(f"oma ratio {r2[i]:.3f} a64 {a64[i]:.6e} oma32 {oma32[i]:.6e} oma64 {oma64[i]:.6e} eps_oma {eps_oma[i]:.2e} o {o[i]}")
print("median eps", np.median(eps))
