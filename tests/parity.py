"""Shared parity checks: the north-star bar (BASELINE.json) as assertions.

Discrete outputs are bit-exact (ids, tile lists, contributor lists); colour
outputs are within max-abs 1e-3 with PSNR >= 60 dB against the reference image.
Depths (the fp64 plane crossings) are checked to 1e-12 relative; weights to 1e-4
relative: display frames take alpha from the certified fp32 kernel value (relative
error bound ~3e-6, nx_fastmath.cuh cert_alpha) — frames that keep the backward state,
and NX_CERTIFIED=0, take it in fp64 (1e-13).
"""
import numpy as np

RGB_TOL = 1e-3       # north star: RGB/alpha max-abs 1e-3
PSNR_MIN = 60.0      # north star: PSNR >= 60 dB vs the reference image
DEPTH_RTOL = 1e-12   # plane crossings: fp64 with the reference's formulas
WEIGHT_RTOL = 1e-4   # certified fp32 alpha (display frames); fp64 paths are at ~1e-13


def psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse)


def compare_frames(gpu, ref, *, rgb_tol=RGB_TOL, check_psnr=True):
    """gpu: DeviceFrame download (device dtypes); ref: fp64 FrameBuffers-like."""
    rep = {}
    assert gpu.ids.shape == ref.ids.shape
    mism = int(np.count_nonzero(gpu.ids != ref.ids))
    rep["ids_mismatch"] = mism
    assert mism == 0, f"{mism} slot ids differ"
    occupied = ref.ids >= 0
    for k, tol in (("depths", DEPTH_RTOL), ("weights", WEIGHT_RTOL)):
        a, b = getattr(gpu, k), getattr(ref, k)
        err = np.abs(a - b)
        rep[k] = float(err.max()) if err.size else 0.0
        rel = err / np.maximum(np.abs(b), 1e-300)
        rep[k + "_rel"] = float(rel[occupied].max()) if occupied.any() else 0.0
        assert np.all(err <= tol * np.maximum(np.abs(b), 1e-12) + 1e-15), f"{k} max err {rep[k]}"
        assert np.all(a[~occupied] == 0.0)
    r = np.abs(gpu.residual.astype(np.float64) - ref.residual)
    rep["residual"] = float(r.max()) if r.size else 0.0
    assert rep["residual"] <= 1e-5
    for k in ("base", "texture", "final_img"):
        a, b = getattr(gpu, k).astype(np.float64), getattr(ref, k)
        rep[k] = float(np.abs(a - b).max()) if a.size else 0.0
        assert rep[k] <= rgb_tol, f"{k} max-abs {rep[k]} > {rgb_tol}"
    if check_psnr and gpu.final_img.size:
        rep["psnr"] = psnr(gpu.final_img, ref.final_img)
        assert rep["psnr"] >= PSNR_MIN, f"PSNR {rep['psnr']:.1f} dB"
    return rep


def is_subsequence(sub, full):
    it = iter(full.tolist())
    return all(x in it for x in sub.tolist())


# render_backward: the reference accumulates in fp64 in a fixed order; the device path
# takes the geometric chain in fp64 but colours (SH, texture) in fp32 and sums with
# fp64 atomics, so gradients agree to ~1e-7 of each array's scale. The bar below is
# GRAD_TOL of the array's largest magnitude, per gradient group.
GRAD_TOL = 1e-5
# The reference field shape takes the tensor-core field backward: MLP products from
# bf16 operands with the 3-term split (relative error <= ~2^-16 per product, fp32
# accumulation) while every ReLU / clamp mask is decided like the reference (exact
# fp32 forward, fp64 re-decision of ambiguous slots). Field-driven gradients then agree
# to a few 1e-5 of each array's scale.
GRAD_TOL_TC = 5e-5
GROUPS = {"mu": slice(0, 3), "quat": slice(3, 7), "log_scale": slice(7, 9), "opacity": slice(9, 10),
          "gamma": slice(10, 12), "sh": slice(12, 60)}


def compare_grads(gpu, ref, tol=GRAD_TOL):
    """gpu / ref: (prims (N,60), table, w1, w2, w3[, blended_error]). Returns the
    per-group normwise errors and asserts each is <= tol."""
    rep = {}
    pairs = {f"prims.{k}": (gpu[0][:, s], ref[0][:, s]) for k, s in GROUPS.items()}
    for i, k in enumerate(("table", "w1", "w2", "w3"), start=1):
        pairs[k] = (gpu[i], ref[i])
    if len(gpu) > 5 and gpu[5] is not None and ref[5] is not None:
        pairs["blended_error"] = (gpu[5], ref[5])
    bad = []
    for k, (a, b) in pairs.items():
        scale = float(np.abs(b).max()) if b.size else 0.0
        err = float(np.abs(a - b).max()) if a.size else 0.0
        rep[k] = (err / scale) if scale > 0 else err
        assert np.all(np.isfinite(a)), f"{k}: non-finite gradients"
        if not (rep[k] <= tol or err <= 1e-12):
            bad.append(f"{k}: max err {err:.3e} vs scale {scale:.3e}")
    assert not bad, "; ".join(bad) + " | " + str({k: f"{v:.1e}" for k, v in rep.items()})
    return rep
