"""GPU: the binning primitives on their own — the one-sweep stable LSD radix sort
(nx_sort.cu) that orders primitives by (depth, id) and keys by tile (the reference's
std::stable_sort / per-tile push_back order, renderer.cpp:102-110), and the single-pass
exclusive scan behind the offsets — against numpy's stable argsort and cumsum, on
adversarial inputs: heavy duplicates, one repeated key (every pass trivial), counts that
are not a multiple of the tile, a device count below the launch capacity (the frame's
sorts run on the grow-only capacity), and the orderable-double depth keys."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2512_13796_b200 import _abi


def _sort(keys, vals, begin, end, cap=None):
    keys = np.ascontiguousarray(keys).copy()
    vals = np.ascontiguousarray(vals, np.uint32).copy()
    n = keys.size
    st = _abi.load().nx_debug_radix_sort(keys.dtype.itemsize, keys.ctypes.data_as(_abi.P),
                                         vals.ctypes.data_as(_abi.PI32), n, cap if cap is not None else n, begin, end)
    assert st == 0
    return keys, vals


def _expect(keys, vals, begin, end):
    k = keys.astype(np.uint64)
    digit = (k >> np.uint64(begin)) & np.uint64((1 << (end - begin)) - 1) if end - begin < 64 else k
    order = np.argsort(digit, kind="stable")
    return keys[order], np.asarray(vals, np.uint32)[order]


def _depth_keys(d):
    """The preprocess's orderable encoding of a double (nx_preprocess.cu depth_key)."""
    b = np.ascontiguousarray(d, np.float64).view(np.uint64)
    neg = (b >> np.uint64(63)) == 1
    return np.where(neg, ~b, b | np.uint64(1 << 63))


@pytest.mark.parametrize("n,cap", [(1, 1), (2, 5000), (2047, 2047), (2049, 4096), (180_000, 400_000),
                                   (1_000_003, 1_000_003)])
def test_u64_depth_sort_matches_stable_argsort(n, cap):
    rng = np.random.default_rng(n)
    # depths in [1, 30] with runs of exact duplicates and near-duplicates (1 ulp apart)
    d = rng.uniform(1.0, 30.0, n)
    d[rng.integers(0, n, n // 5)] = d[rng.integers(0, n, n // 5)]
    nb = rng.integers(0, n, n // 10)
    d[nb] = np.nextafter(d[nb], 2.0 * d[nb])
    keys = _depth_keys(d)
    vals = np.arange(n, dtype=np.uint32)
    got_k, got_v = _sort(keys, vals, 0, 64, cap)
    want_k, want_v = _expect(keys, vals, 0, 64)
    assert np.array_equal(got_k, want_k) and np.array_equal(got_v, want_v)
    # the (depth, id) order the reference's stable sort gives
    assert np.array_equal(got_v, np.lexsort((np.arange(n), d)).astype(np.uint32))


@pytest.mark.parametrize("n,bits", [(3_000_001, 15), (2_000_000, 13), (65_537, 8), (10, 3)])
def test_u32_tile_sort_matches_stable_argsort(n, bits):
    rng = np.random.default_rng(bits)
    keys = rng.integers(0, 1 << bits, n, dtype=np.uint32)
    keys[: n // 3] = np.sort(keys[: n // 3])  # long already-sorted runs, as the emit order gives
    vals = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    got_k, got_v = _sort(keys, vals, 0, bits, cap=n + 12345)
    want_k, want_v = _expect(keys, vals, 0, bits)
    assert np.array_equal(got_k, want_k) and np.array_equal(got_v, want_v)


def test_single_key_every_pass_trivial():
    n = 50_000
    keys = np.full(n, 0x0123456789abcdef, np.uint64)
    vals = np.arange(n, dtype=np.uint32)[::-1].copy()
    got_k, got_v = _sort(keys, vals, 0, 64)
    assert np.array_equal(got_k, keys) and np.array_equal(got_v, vals)


def test_partial_bit_range_sorts_on_those_bits_only():
    rng = np.random.default_rng(5)
    n = 100_000
    keys = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint32)
    got_k, got_v = _sort(keys, vals, 24, 40)
    want_k, want_v = _expect(keys, vals, 24, 40)
    assert np.array_equal(got_k, want_k) and np.array_equal(got_v, want_v)


@pytest.mark.parametrize("n,cap", [(1, 1), (4095, 4095), (4097, 9000), (400_000, 400_000), (300_000, 1_000_000)])
def test_scan_matches_cumsum(n, cap):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 50, n, dtype=np.int32)
    x[rng.integers(0, n, n // 4)] = 0
    out = np.empty(n, np.int32)
    total = np.zeros(1, np.int32)
    lib = _abi.load()
    assert lib.nx_debug_scan(x.ctypes.data_as(_abi.PI32), out.ctypes.data_as(_abi.PI32), n, cap,
                             total.ctypes.data_as(_abi.PI32)) == 0
    want = np.concatenate([[0], np.cumsum(x[:-1], dtype=np.int64)]).astype(np.int32)
    assert np.array_equal(out, want)
    assert int(total[0]) == int(x.sum())
