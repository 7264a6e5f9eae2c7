// Exact, order-independent accumulation for render_backward's reductions.
//
// The reference's backward is bit-stable for any worker count (threading.hpp:12-16;
// test_train.cpp "training is deterministic run to run"): it reduces per-tile /
// per-worker partials in a fixed order. On the GPU the partials meet in atomics,
// whose order varies run to run, and floating-point addition does not commute
// bit-exactly. Here every addend is instead cut into 32-bit chunks of one fixed-point
// number (lsb 2^kXaccE0) and each chunk is added to an int64 word with an integer
// atomic. Integer addition commutes, so the words — and the value read back from them —
// are the same whatever the order; the sum is exact (no rounding until the single
// read-back), which is at least as accurate as any ordered fp64 sum.
//
// Layout: value i of an accumulator with m values owns words w[k * m + i] for
// k < kXaccWords, plus a flags word w[kXaccWords * m + i] (+inf / -inf / NaN addends).
// Range: the bits of an addend below 2^kXaccE0 (~2.9e-39) are dropped (toward zero), so
// fp32 addends above 2^-104 and fp64 addends above 2^-75 (~2.6e-23) keep every bit;
// fp32 addends up to 2^55 and fp64 addends up to 2^52 fit, larger ones saturate to +-inf.
// Each word takes < 2^32 per addend, so 2^31 addends per value cannot overflow it.
// Readers (xacc_take) zero what they read: accumulators stay zero between uses.
#pragma once
#include <cstdint>

namespace nx {

constexpr int kXaccWords = 6;
constexpr int kXaccE0 = -128;
constexpr int kXaccWordsTotal = kXaccWords + 1;  // + flags

enum : unsigned long long { kXaccPosInf = 1, kXaccNegInf = 2, kXaccNaN = 4 };

struct Xacc {
    unsigned long long* w;
    int64_t m;  // number of values
};

inline size_t xacc_bytes(int64_t m) { return static_cast<size_t>(m) * kXaccWordsTotal * sizeof(unsigned long long); }

#ifdef __CUDACC__
__device__ __forceinline__ void xacc_chunk(const Xacc& x, int64_t i, int k, unsigned long long c, bool neg) {
    if (c) atomicAdd(x.w + k * x.m + i, neg ? (0ull - c) : c);
}
__device__ __forceinline__ void xacc_special(const Xacc& x, int64_t i, unsigned long long f) {
    atomicOr(x.w + kXaccWords * x.m + i, f);
}

// fp32 addend: 24-bit significand -> at most two chunks. The common case (a normal
// number inside the range) is a dozen instructions inline; zero / subnormal / tiny /
// huge / non-finite addends take the out-of-line path.
static __device__ __noinline__ void xacc_add_f32_slow(const Xacc& x, int64_t i, float v) {
    const uint32_t b = __float_as_uint(v);
    const int ex = static_cast<int>((b >> 23) & 0xff);
    const bool neg = b >> 31;
    if (ex == 0xff) {
        xacc_special(x, i, (b & 0x7fffff) ? kXaccNaN : neg ? kXaccNegInf : kXaccPosInf);
        return;
    }
    uint64_t m = b & 0x7fffffu;
    if (ex) m |= 0x800000u;
    if (!m) return;
    int s = (ex ? ex : 1) - 150 - kXaccE0;  // lsb position above 2^E0
    if (s < 0) {
        if (s <= -24) return;
        m >>= -s;
        s = 0;
        if (!m) return;
    }
    const int k = s >> 5, r = s & 31;
    if (k + 1 >= kXaccWords) {
        xacc_special(x, i, neg ? kXaccNegInf : kXaccPosInf);
        return;
    }
    const uint64_t y = m << r;
    xacc_chunk(x, i, k, y & 0xffffffffull, neg);
    xacc_chunk(x, i, k + 1, y >> 32, neg);
}

__device__ __forceinline__ void xacc_add(const Xacc& x, int64_t i, float v) {
    const uint32_t b = __float_as_uint(v);
    const int s = static_cast<int>((b >> 23) & 0xff) - 150 - kXaccE0;
    const int k = s >> 5;
    if (s < 0 || k + 1 >= kXaccWords || ((b >> 23) & 0xff) == 0) {  // zero / subnormal / out of range / inf / NaN
        if (b << 1) xacc_add_f32_slow(x, i, v);
        return;
    }
    const uint64_t y = static_cast<uint64_t>((b & 0x7fffffu) | 0x800000u) << (s & 31);  // < 2^56
    const uint64_t lo = y & 0xffffffffull, hi = y >> 32;
    const bool neg = b >> 31;
    if (lo) atomicAdd(x.w + k * x.m + i, neg ? (0ull - lo) : lo);
    if (hi) atomicAdd(x.w + (k + 1) * x.m + i, neg ? (0ull - hi) : hi);
}

// fp64 addend: 53-bit significand -> at most three chunks.
__device__ __forceinline__ void xacc_add(const Xacc& x, int64_t i, double v) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    const int ex = static_cast<int>((b >> 52) & 0x7ff);
    const bool neg = b >> 63;
    if (ex == 0x7ff) {
        xacc_special(x, i, (b & 0xfffffffffffffull) ? kXaccNaN : neg ? kXaccNegInf : kXaccPosInf);
        return;
    }
    uint64_t m = b & 0xfffffffffffffull;
    if (ex) m |= 1ull << 52;
    if (!m) return;
    int s = (ex ? ex : 1) - 1075 - kXaccE0;
    if (s < 0) {
        if (s <= -53) return;
        m >>= -s;
        s = 0;
        if (!m) return;
    }
    const int k = s >> 5, r = s & 31;
    const uint64_t lo = m << r, hi = r ? (m >> (64 - r)) : 0ull;
    const int top = hi ? k + 2 : k + 1;
    if (top >= kXaccWords) {
        xacc_special(x, i, neg ? kXaccNegInf : kXaccPosInf);
        return;
    }
    xacc_chunk(x, i, k, lo & 0xffffffffull, neg);
    xacc_chunk(x, i, k + 1, lo >> 32, neg);
    xacc_chunk(x, i, k + 2, hi, neg);
}

// Reads value i (exact sum, rounded once — to within a couple of ulp — by a fixed
// sequence of operations) and zeroes its words.
__device__ __forceinline__ double xacc_take(const Xacc& x, int64_t i) {
    unsigned long long* flag = x.w + kXaccWords * x.m + i;
    const unsigned long long f = *flag;
    int64_t wv[kXaccWords];
    bool any = false;
#pragma unroll
    for (int k = 0; k < kXaccWords; ++k) {
        wv[k] = static_cast<int64_t>(x.w[k * x.m + i]);
        any |= wv[k] != 0;
    }
    if (any) {
#pragma unroll
        for (int k = 0; k < kXaccWords; ++k) x.w[k * x.m + i] = 0ull;
    }
    if (f) {
        *flag = 0ull;
        if ((f & kXaccNaN) || ((f & kXaccPosInf) && (f & kXaccNegInf))) return __longlong_as_double(0x7ff8000000000000ll);
        return (f & kXaccPosInf) ? __longlong_as_double(0x7ff0000000000000ll)
                                 : __longlong_as_double(static_cast<long long>(0xfff0000000000000ull));
    }
    if (!any) return 0.0;
    // carry-normalise into 32-bit digits + a signed top
    uint32_t d[kXaccWords];
    int64_t c = 0;
#pragma unroll
    for (int k = 0; k < kXaccWords; ++k) {
        const int64_t t = wv[k] + c;
        d[k] = static_cast<uint32_t>(t);
        c = (t - static_cast<int64_t>(d[k])) >> 32;
    }
    const bool neg = c < 0;
    if (neg) {  // magnitude: two's complement of the (kXaccWords + 1)-digit number
        uint64_t carry = 1;
#pragma unroll
        for (int k = 0; k < kXaccWords; ++k) {
            const uint64_t t = static_cast<uint64_t>(~d[k]) + carry;
            d[k] = static_cast<uint32_t>(t);
            carry = t >> 32;
        }
        c = ~c + static_cast<int64_t>(carry);
    }
    // sum of non-negative terms from the top (scale 2^(E0 + 32 k))
    double r = static_cast<double>(c) * 0x1p64;  // 2^(E0 + 32 * kXaccWords) = 2^64
    constexpr double kScale[kXaccWords] = {0x1p-128, 0x1p-96, 0x1p-64, 0x1p-32, 0x1p0, 0x1p32};
#pragma unroll
    for (int k = kXaccWords - 1; k >= 0; --k) r += static_cast<double>(d[k]) * kScale[k];
    return neg ? -r : r;
}
#endif

static_assert(kXaccE0 + 32 * kXaccWords == 64, "xacc_take's top scale");

}  // namespace nx
