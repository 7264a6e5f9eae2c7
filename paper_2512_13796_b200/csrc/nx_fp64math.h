// fp64 exp / log for the compositing hot loop (eval_kernel / axis_power,
// kernel.hpp:16-30), written for the sm_100a issue budget: polynomial
// coefficients are read from the constant bank as direct DFMA operands (no
// per-call register materialisation, which dominates the CUDA math library's
// exp/log in this loop), and only the argument ranges the kernel can produce take
// the fast path. Accuracy: <= 1 ulp-class (checked against glibc over 1e7
// samples by tests/test_fp64math.py); the reference's own glibc exp/log are
// within 1 ulp as well, so decisions agree away from ~1e-15-relative ties (the
// measured margins are >= 1e-9).
//
// Host-compilable (g++) so that the CPU test exercises the very same code.
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define NX_FM_HD __host__ __device__ __forceinline__
#define NX_FM_CONST __constant__
#else
#define NX_FM_HD static inline
#define NX_FM_CONST static const
#endif

namespace nx {
namespace fm {

// 1/k! for e^r on |r| <= ln2/2 (degree 14: truncation r^15/15! < 2^-63 relative)
NX_FM_CONST double kExpC[15] = {1.0,
                                1.0,
                                0.5,
                                0.16666666666666666,
                                0.041666666666666664,
                                0.008333333333333333,
                                0.001388888888888889,
                                1.984126984126984e-4,
                                2.48015873015873e-5,
                                2.7557319223985893e-6,
                                2.755731922398589e-7,
                                2.505210838544172e-8,
                                2.08767569878681e-9,
                                1.6059043836821613e-10,
                                1.1470745597729725e-11};
// 2/(2k+1) for log(1+f) = 2 atanh(s) = sum 2 s^(2k+1)/(2k+1), |s| <= 0.1716
NX_FM_CONST double kLogC[12] = {2.0,
                                0.6666666666666666,
                                0.4,
                                0.2857142857142857,
                                0.2222222222222222,
                                0.18181818181818182,
                                0.15384615384615385,
                                0.13333333333333333,
                                0.11764705882352941,
                                0.10526315789473684,
                                0.09523809523809523,
                                0.08695652173913043};

NX_FM_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

NX_FM_HD uint64_t as_u64(double x) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
NX_FM_HD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

// e^x. Fast path for x in [-708, 709]; outside it defers to the library exp.
NX_FM_HD double exp64(double x) {
    if (!(x >= -708.0 && x <= 709.0)) return exp(x);
    const double kLog2e = 1.4426950408889634;
    const double kLn2Hi = 6.93147180369123816490e-01;  // fdlibm split
    const double kLn2Lo = 1.90821492927058770002e-10;
    const double k = rint(x * kLog2e);
    const double r0 = fma_(-k, kLn2Hi, x);  // exact: ln2_hi has 21 trailing zero bits
    const double r = fma_(-k, kLn2Lo, r0);
    const double rlo = fma_(-k, kLn2Lo, r0 - r);  // rounding error of r (r0 - r is exact)
    // e^r = 1 + r + r^2 q(r), q = 1/2 + r/6 + ...; the small terms absorb the errors
    double q = kExpC[14];
#pragma unroll
    for (int i = 13; i >= 2; --i) q = fma_(q, r, kExpC[i]);
    const double s = fma_(r * r, q, rlo);
    const double p = 1.0 + (r + s);
    // scale by 2^k: k in [-1022, 1023] for the fast-path range, except the low end
    const int ki = static_cast<int>(k);
    if (ki < -1020) return p * as_f64(static_cast<uint64_t>(ki + 1023 + 100) << 52) * 7.888609052210118e-31;  // 2^-100
    return p * as_f64(static_cast<uint64_t>(ki + 1023) << 52);
}

// ln x. Fast path for finite normal x > 0; otherwise the library log.
NX_FM_HD double log64(double x) {
    const uint64_t u = as_u64(x);
    const uint64_t ex = (u >> 52) & 0x7ff;
    if (!(x > 0.0) || ex == 0 || ex == 0x7ff) return log(x);
    // x = m 2^e with m in [sqrt(1/2), sqrt(2))
    int e = static_cast<int>(ex) - 1023;
    uint64_t mu = (u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
    double m = as_f64(mu);
    if (m > 1.4142135623730951) {
        m *= 0.5;
        e += 1;
    }
    // fdlibm-style reduction (e_log.c): ln(1+f) = f - (hfsq - s (hfsq + R)), R ~ odd
    // atanh tail in s = f/(2+f), so the leading term f is exact and the rounding
    // errors sit in the small correction.
    const double f = m - 1.0;  // exact (Sterbenz)
    const double s = f / (2.0 + f);
    const double z = s * s;
    double R = kLogC[11];
#pragma unroll
    for (int i = 10; i >= 1; --i) R = fma_(R, z, kLogC[i]);
    R = R * z;  // = 2/3 z + 2/5 z^2 + ... (the series of 2 atanh(s)/s - 2, times 1/2 * ... see below)
    // 2 atanh(s) = 2s + s*R  and  f = 2s + s*f  =>  ln(1+f) = f - s*(f - R)
    const double lm = f - s * (f - R);
    const double kLn2Hi = 6.93147180369123816490e-01;
    const double kLn2Lo = 1.90821492927058770002e-10;
    const double de = static_cast<double>(e);
    return fma_(de, kLn2Hi, fma_(de, kLn2Lo, lm));
}

// axis_power / eval_kernel (kernel.hpp:16-30) on the fast transcendentals.
NX_FM_HD double axis_power(double u, double g) {
    if (u == 0.0) return 0.0;
    if (g == 1.0) return u * u;
    const double e = 2.0 * g * log64(fabs(u));
    if (e > 700.0) return INFINITY;
    return exp64(e);
}
NX_FM_HD double eval_kernel(double u, double v, double o, double gx, double gy) {
    const double p = axis_power(u, gx) + axis_power(v, gy);
    if (isinf(p)) return 0.0;
    return o * exp64(-0.5 * p);
}

}  // namespace fm
}  // namespace nx
