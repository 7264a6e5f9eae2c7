"""GPU: the table-driven fp64 exp / log of the compositing kernels (nx_fastmath.cuh)
against the C library's (glibc: what the reference's kernel.hpp:16-30 calls), in ulps,
over the argument ranges the kernel evaluates — ln|u| for |u| in (2^-40, 8], exp of the
axis-power exponents 2 g ln|u| in [-700, 700] and of the kernel's -p/2 in [-700, 0] — plus
the special values that take the library path."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2512_13796_b200 as nx
from paper_2512_13796_b200 import _abi


def _run(fn, x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    st = _abi.load().nx_debug_fastmath(fn, x.ctypes.data_as(_abi.PD), y.ctypes.data_as(_abi.PD), x.size)
    assert st == 0
    return y


def _ulp_err(got, want):
    want = np.asarray(want)
    fin = np.isfinite(want) & (want != 0)
    ulp = np.spacing(np.abs(want[fin]))
    return float(np.max(np.abs(got[fin] - want[fin]) / ulp)) if fin.any() else 0.0


def _libm(f, x):
    return np.array([f(v) for v in x.tolist()])  # CPython's math module calls the C library


def test_fast_log_within_2_ulp_of_libm():
    rng = np.random.default_rng(11)
    x = np.concatenate([np.exp(rng.uniform(math.log(2.0 ** -40), math.log(8.0), 1_000_000)),
                        rng.uniform(0.9, 1.1, 500_000), rng.uniform(0.0, 3.0, 500_000),
                        np.array([1.0, 2.0, 0.5, 1.0 + 2 ** -52, 1.0 - 2 ** -53, 1.5, 1.0078125])])
    x = x[x > 0]
    got = _run(0, x)
    want = _libm(math.log, x)
    # near x = 1 the result is small, so relative ulps are not the measure that matters
    # (ln|u| feeds exp(2 g ln|u|)): check the absolute error there, ulps elsewhere
    far = np.abs(x - 1.0) > 0.25
    assert _ulp_err(got[far], want[far]) <= 2.0
    assert float(np.max(np.abs(got - want))) <= 4e-16 * np.maximum(1.0, np.abs(want)).max()
    print(f"fast log: max {_ulp_err(got[far], want[far]):.2f} ulp away from 1, "
          f"max abs err {np.max(np.abs(got - want)):.2e}")


def test_fast_exp_within_2_ulp_of_libm():
    rng = np.random.default_rng(12)
    x = np.concatenate([rng.uniform(-700.0, 700.0, 1_000_000), rng.uniform(-8.0, 3.0, 1_000_000),
                        rng.uniform(-1e-3, 1e-3, 100_000),
                        np.array([0.0, -0.0, 1.0, -1.0, 707.9, -707.9, math.log(2.0), 1e-300])])
    got = _run(1, x)
    want = _libm(math.exp, x)
    err = _ulp_err(got, want)
    assert err <= 2.0, err
    print(f"fast exp: max {err:.2f} ulp")


def test_special_values_take_the_library_path():
    x = np.array([0.0, 5e-324, 1e-310, np.inf, np.nan, -1.0])
    got = _run(0, x)
    ref = _run(2, x)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    fin = ~np.isnan(ref)
    assert np.array_equal(got[fin], ref[fin])
    x = np.array([-750.0, -708.5, 709.5, 800.0, np.inf, -np.inf, np.nan])
    got = _run(1, x)
    ref = _run(3, x)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    fin = ~np.isnan(ref)
    assert np.array_equal(got[fin], ref[fin])



def test_certified_fp32_alpha_bounds_hold():
    """cert_alpha (nx_fastmath.cuh): the SFU fp32 kernel value and 1 - alpha against the
    fp64 routine over 3M samples spanning the kernel's argument ranges (|u|, |v| up to the
    support radius, gamma 1..6, opacity 0.004..0.999): the error never exceeds the
    certified bound, and the bound stays tight enough (median < 2e-5 relative)."""
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
    assert np.all(np.abs(a32 - a64) <= eps * np.maximum(a64, 1e-30) + 1e-30)
    oma64 = 1.0 - a64
    ok = oma64 > 1e-6
    assert np.all(np.abs(oma32[ok] - oma64[ok]) <= eps_oma[ok] * oma64[ok])
    near = np.abs(a64 - 1 / 255) < 0.5 / 255
    print(f"cert alpha: median bound {np.median(eps):.2e}, near-threshold median {np.median(eps[near]):.2e}, "
          f"max error/bound {np.max(np.abs(a32 - a64) / (eps * np.maximum(a64, 1e-30))):.3f}")
    assert np.median(eps) < 2e-5
