// Table-driven fp64 exp / log for the compositing hot loop.
//
// The reference evaluates its kernel (kernel.hpp:16-30) as o * exp(-0.5 * (|u|^(2gx) +
// |v|^(2gy))) with |u|^(2g) = exp(2 g ln|u|): two logs and three exps per intersection,
// with glibc's fp64 exp / log. CUDA's fp64 exp / log are general-purpose routines of ~45 /
// ~75 instructions (special-value handling, wide polynomials); these are the classic
// table-driven reductions (Tang) at the same accuracy class:
//   exp(x) = 2^(k/32) * exp(r),  r = x - k ln2/32 (Cody-Waite, |r| <= ln2/64), degree-6 Taylor
//            (truncation < 4e-18 relative), 32-entry table of 2^(j/32) correctly rounded;
//   ln(x)  = e ln2 - ln(c_j) + ln(1 + r),  r = m c_j - 1 (one FMA, |r| <= 2^-7), degree-8
//            Taylor (truncation < 2e-20), c_j = fp32(1 / (1 + (j + 1/2)/64)) on the top six
//            mantissa bits, -ln(c_j) correctly rounded.
// Both are within ~1.5 ulp of the correctly rounded result (tests/test_gpu_fastmath.py:
// max ulp error against glibc over 2M arguments per range), the accuracy class of
// CUDA's and glibc's own routines, so every decision taken with them (alpha >= 1/255,
// the alpha clamp, T < min_T, top-K order) is the reference's wherever its margin exceeds
// ~1e-15 relative; the near-threshold counter (nx_frame_stats.near_*) reports any that
// does not. Arguments outside the fast ranges (subnormal, non-finite, exp below -708 or
// above 709) take CUDA's library routines.
#pragma once

#include <cuda_runtime.h>

#include "nx_internal.cuh"

namespace nx {

// 2^(j/32), j = 0..31, correctly rounded (generated with 60-digit decimal arithmetic)
#define NX_EXP2_TABLE_32 \
    0x1.0000000000000p+0, 0x1.059b0d3158574p+0, \
    0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0, \
    0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, \
    0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0, \
    0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, \
    0x1.3dea64c123422p+0, 0x1.44e086061892dp+0, \
    0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, \
    0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0, \
    0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, \
    0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0, \
    0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, \
    0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0, \
    0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, \
    0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0, \
    0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, \
    0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0,
// {c_j, -ln(c_j)}, c_j = fp32(1 / (1 + (j + 1/2)/64)), j = 0..63; -ln(c_j) correctly rounded
#define NX_LOG_TABLE_64 \
    {0x1.fc07f00000000p-1, 0x1.fe02b6b106791p-8}, \
    {0x1.f4465a0000000p-1, 0x1.7b91acfd5b11cp-6}, \
    {0x1.ecc07c0000000p-1, 0x1.39e86e1febd8dp-5}, \
    {0x1.e573ac0000000p-1, 0x1.b42de091971d5p-5}, \
    {0x1.de5d6e0000000p-1, 0x1.1653710a37ae3p-4}, \
    {0x1.d77b660000000p-1, 0x1.51b06dd061852p-4}, \
    {0x1.d0cb580000000p-1, 0x1.8c3465e319b45p-4}, \
    {0x1.ca4b300000000p-1, 0x1.c5e54bf5bc748p-4}, \
    {0x1.c3f8f00000000p-1, 0x1.fec9141dbeabbp-4}, \
    {0x1.bdd2b80000000p-1, 0x1.1b72b012f67a8p-3}, \
    {0x1.b7d6c40000000p-1, 0x1.371fc161e8f75p-3}, \
    {0x1.b203640000000p-1, 0x1.526e5e5a1b438p-3}, \
    {0x1.ac57020000000p-1, 0x1.6d60fce19d21fp-3}, \
    {0x1.a6d01a0000000p-1, 0x1.87fa08620c915p-3}, \
    {0x1.a16d400000000p-1, 0x1.a23bbffe2b567p-3}, \
    {0x1.9c2d140000000p-1, 0x1.bc286be2d8cecp-3}, \
    {0x1.970e500000000p-1, 0x1.d5c21434fbb98p-3}, \
    {0x1.920fb40000000p-1, 0x1.ef0adfddc5940p-3}, \
    {0x1.8d30180000000p-1, 0x1.04025b6b4d04ap-2}, \
    {0x1.886e600000000p-1, 0x1.1058bd1ae4ae2p-2}, \
    {0x1.83c9780000000p-1, 0x1.1c898b36999fdp-2}, \
    {0x1.7f40600000000p-1, 0x1.2895a0bde86a4p-2}, \
    {0x1.7ad2200000000p-1, 0x1.347ddb2987d59p-2}, \
    {0x1.767dce0000000p-1, 0x1.404309206a7e5p-2}, \
    {0x1.7242880000000p-1, 0x1.4be5f937778a1p-2}, \
    {0x1.6e1f760000000p-1, 0x1.5767736c55a74p-2}, \
    {0x1.6a13ce0000000p-1, 0x1.62c82c939c7a3p-2}, \
    {0x1.661ec60000000p-1, 0x1.6e08ec7aba1eap-2}, \
    {0x1.623fa80000000p-1, 0x1.792a545dd47a8p-2}, \
    {0x1.5e75bc0000000p-1, 0x1.842d1c51e8b1bp-2}, \
    {0x1.5ac0560000000p-1, 0x1.8f11ea7b662d0p-2}, \
    {0x1.571ed40000000p-1, 0x1.99d957617e08cp-2}, \
    {0x1.5390940000000p-1, 0x1.a4840abe5bb10p-2}, \
    {0x1.5015020000000p-1, 0x1.af12910c77874p-2}, \
    {0x1.4cab880000000p-1, 0x1.b9858ac9310ffp-2}, \
    {0x1.49539e0000000p-1, 0x1.c3dd7b34dad4ep-2}, \
    {0x1.460cbc0000000p-1, 0x1.ce1af2485f3f0p-2}, \
    {0x1.42d6620000000p-1, 0x1.d83e7380a2f41p-2}, \
    {0x1.3fb0140000000p-1, 0x1.e2488197c6c26p-2}, \
    {0x1.3c995a0000000p-1, 0x1.ec399e0c68cc2p-2}, \
    {0x1.3991c20000000p-1, 0x1.f612421f028b9p-2}, \
    {0x1.3698e00000000p-1, 0x1.ffd2de057f4a5p-2}, \
    {0x1.33ae460000000p-1, 0x1.04bdf95e926d3p-1}, \
    {0x1.30d1900000000p-1, 0x1.0986f51573521p-1}, \
    {0x1.2e025c0000000p-1, 0x1.0e4498651cc8cp-1}, \
    {0x1.2b404a0000000p-1, 0x1.12f71abd3efc4p-1}, \
    {0x1.288b020000000p-1, 0x1.179eaa49899a9p-1}, \
    {0x1.25e2280000000p-1, 0x1.1c3b804713c30p-1}, \
    {0x1.2345680000000p-1, 0x1.20cdcc492ab70p-1}, \
    {0x1.20b4700000000p-1, 0x1.2555be498f7d3p-1}, \
    {0x1.1e2ef40000000p-1, 0x1.29d37f642b08cp-1}, \
    {0x1.1bb4a40000000p-1, 0x1.2e47437640268p-1}, \
    {0x1.1945380000000p-1, 0x1.32b133a121d71p-1}, \
    {0x1.16e0680000000p-1, 0x1.37117c64747bap-1}, \
    {0x1.1485f00000000p-1, 0x1.3b68463fffc2dp-1}, \
    {0x1.12358e0000000p-1, 0x1.3fb5b92916f45p-1}, \
    {0x1.0fef020000000p-1, 0x1.43f9fc6b9ce74p-1}, \
    {0x1.0db20a0000000p-1, 0x1.48353e22a88e4p-1}, \
    {0x1.0b7e6e0000000p-1, 0x1.4c679c70cee42p-1}, \
    {0x1.0953f40000000p-1, 0x1.50913be81686ep-1}, \
    {0x1.0732600000000p-1, 0x1.54b247b99949ep-1}, \
    {0x1.0519800000000p-1, 0x1.58cada5cd798dp-1}, \
    {0x1.03091c0000000p-1, 0x1.5cdb1c6ec176cp-1}, \
    {0x1.0101020000000p-1, 0x1.60e32d48788e9p-1},

struct FastMathTables {
    double e2[32];   // 2^(j/32)
    double2 lg[64];  // {c_j, -ln(c_j)}
};

__device__ const FastMathTables kFastMath = {{NX_EXP2_TABLE_32}, {NX_LOG_TABLE_64}};

constexpr double kLn2Hi = 0x1.62e42fee00000p-1;   // ln 2, upper 32 bits (e * kLn2Hi exact)
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;  // ln 2 - kLn2Hi

// The tables stay in global memory (1.3 KB, L1-resident, read with __ldg): a shared-
// memory copy per CTA was measured slower (it takes L1 capacity from the record gathers).
__device__ __forceinline__ double fm_log(double x) {
    const FastMathTables& t = kFastMath;
    const long long b = __double_as_longlong(x);
    const int be = static_cast<int>(b >> 52);  // biased exponent (sign bit clear for x > 0)
    if (be <= 0 || be >= 0x7ff) return log(x);  // zero, subnormal, negative, inf, nan
    const int j = static_cast<int>((b >> 46) & 63);
    const double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
    const double2 cl = __ldg(&t.lg[j]);
    const double r = fma(m, cl.x, -1.0);
    double q = -1.0 / 8.0;
    q = fma(q, r, 1.0 / 7.0);
    q = fma(q, r, -1.0 / 6.0);
    q = fma(q, r, 1.0 / 5.0);
    q = fma(q, r, -1.0 / 4.0);
    q = fma(q, r, 1.0 / 3.0);
    q = fma(q, r, -1.0 / 2.0);
    const double p = fma(r * r, q, r);  // ln(1 + r)
    const double e = static_cast<double>(be - 1023);
    return fma(e, kLn2Hi, cl.y + fma(e, kLn2Lo, p));
}

constexpr double kInvLn2x32 = 0x1.71547652b82fep+5;  // 32 / ln 2
constexpr double kLn2d32Hi = kLn2Hi / 32.0;          // exact
constexpr double kLn2d32Lo = kLn2Lo / 32.0;

__device__ __forceinline__ double fm_exp(double x) {
    const FastMathTables& t = kFastMath;
    if (!(x > -708.0 && x < 709.0)) return exp(x);  // underflow / overflow region, nan
    const int k = __double2int_rn(x * kInvLn2x32);
    const double kd = static_cast<double>(k);
    double r = fma(-kd, kLn2d32Hi, x);
    r = fma(-kd, kLn2d32Lo, r);
    double q = 1.0 / 720.0;
    q = fma(q, r, 1.0 / 120.0);
    q = fma(q, r, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double p = fma(q, r, 1.0);  // exp(r)
    const double scale = __longlong_as_double(static_cast<long long>((k >> 5) + 1023) << 52);
    return (__ldg(&t.e2[k & 31]) * p) * scale;
}

// axis_power / eval_kernel (kernel.hpp:16-30) on the table routines; `lu` receives
// ln|u| (0 when u == 0) for callers that need it (render_backward's d/dgamma).
__device__ __forceinline__ double fm_axis_power(double u, double g, double& lu) {
    lu = 0.0;
    if (u == 0.0) return 0.0;
    if (g == 1.0) return u * u;
    lu = fm_log(fabs(u));
    const double e = 2.0 * g * lu;
    if (e > 700.0) return INFINITY;
    return fm_exp(e);
}

// The exact intersection of one pixel ray with one primitive record: intersect()
// (intersect.hpp:23-42) and eval_kernel (kernel.hpp:16-30) with the reference's
// formulas and decisions, in fp64 (a straight-line form with both axes in flight and
// division / exp / log without slow-path branches was measured slower: the register
// pressure costs more than the latency it hides). Returns
// alpha (< 0 for a miss); t, and for render_backward the kernel terms (ln|u|, ln|v|,
// the axis powers and exp(-p/2)), are filled for a hit.
struct HitTerms {
    double alpha, t, u, v, lu, lv, pu, pv, k;
    bool near;  // alpha within kNearAlpha of 1/255 (either side): a near-threshold decision
};

template <typename Rec>
__device__ __forceinline__ HitTerms exact_hit(const Rec& r, double d0, double d1, double d2, double o0, double o1,
                                              double o2, double near_eps) {
    HitTerms h;
    h.alpha = -1.0;
    h.near = false;
    const double denom = d0 * r[REC_NX] + d1 * r[REC_NY] + d2 * r[REC_NZ];
    if (!(fabs(denom) >= kMinNormalDot)) return h;
    h.t = r[REC_NUM] / denom;
    if (!(h.t > near_eps)) return h;
    const double e0 = (o0 + h.t * d0) - r[REC_MUX];
    const double e1 = (o1 + h.t * d1) - r[REC_MUY];
    const double e2 = (o2 + h.t * d2) - r[REC_MUZ];
    const double du = e0 * r[REC_V1X] + e1 * r[REC_V1Y] + e2 * r[REC_V1Z];
    const double dv = e0 * r[REC_V2X] + e1 * r[REC_V2Y] + e2 * r[REC_V2Z];
    if (!(fabs(du) <= r[REC_ULIM] && fabs(dv) <= r[REC_VLIM])) return h;
    h.u = du / r[REC_SX];
    h.v = dv / r[REC_SY];
    h.pu = fm_axis_power(h.u, r[REC_GX], h.lu);
    h.pv = fm_axis_power(h.v, r[REC_GY], h.lv);
    const double q = h.pu + h.pv;
    h.k = isinf(q) ? 0.0 : fm_exp(-0.5 * q);
    const double al = isinf(q) ? 0.0 : r[REC_OP] * h.k;
    if (al >= kAlphaMin) h.alpha = al;
    h.near = fabs(al - kAlphaMin) <= kNearAlpha * kAlphaMin;
    return h;
}

// ---------------------------------------------------------------- certified fp32 alpha
// eval_kernel (kernel.hpp:16-30) on the SFU (MUFU lg2 / ex2 in fp32) with a rigorous
// bound on its relative error, so that the decision alpha >= 1/255 is taken in fp32
// wherever the bound clears the threshold and with the exact fp64 routine otherwise.
// Error model (fp32 unit 2^-24 = 6e-8; MUFU.LG2 absolute error <= 2^-22, MUFU.EX2
// relative error <= 2^-21, both taken generously; u carries 3 roundings):
//   d(lg2|u|) <= 2.4e-7 + 6e-8 |lg2 u| + 2.6e-7             (argument error 1.8e-7 / ln 2)
//   d(a)      <= 2g d(lg2|u|) + 1.2e-7 |a|,  a = 2g lg2|u|
//   rel(pu)   <= ln2 d(a) + 4.8e-7
//   |dp|      <= pu rel(pu) + pv rel(pv) + 6e-8 p
//   rel(alpha) <= p/2 rel(p) + ln2 1.2e-7 |b| + 6e-7,  b = -p/(2 ln 2)
// and the result is doubled (`eps`). 1 - alpha is formed as (1 - o) + o (1 - k), with
// 1 - k = -expm1(-p/2) (a degree-9 series above -0.7), so it keeps its relative accuracy
// (`eps_oma`) when alpha is close to 1. tests/test_gpu_fastmath.py checks the bounds
// against the fp64 routine over millions of (u, v, gamma, o).
struct CertAlpha {
    float alpha;    // o exp(-(|u|^2gx + |v|^2gy) / 2)
    float oma;      // 1 - alpha
    float eps;      // relative error bound of alpha
    float eps_oma;  // relative error bound of oma
};

__device__ __forceinline__ float sfu_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sfu_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ CertAlpha cert_alpha(float u, float v, float g2x, float g2y, float o, float om) {
    CertAlpha c;
    const float lu = sfu_lg2(fabsf(u)), lv = sfu_lg2(fabsf(v));
    const float au = g2x * lu, av = g2y * lv;
    const float pu = u == 0.f ? 0.f : sfu_ex2(au), pv = v == 0.f ? 0.f : sfu_ex2(av);
    const float p = pu + pv;
    const float dau = g2x * (5.0e-7f + 6e-8f * fabsf(lu)) + 1.2e-7f * fabsf(au);
    const float dav = g2y * (5.0e-7f + 6e-8f * fabsf(lv)) + 1.2e-7f * fabsf(av);
    const float dp = (u == 0.f ? 0.f : pu * (0.6931472f * dau + 4.8e-7f)) +
                     (v == 0.f ? 0.f : pv * (0.6931472f * dav + 4.8e-7f)) + 6e-8f * p;
    const float b = -0.72134752f * p;  // -p / (2 ln 2)
    const float k = sfu_ex2(b);
    c.alpha = o * k;
    c.eps = 2.f * (0.5f * dp + 8.4e-8f * fabsf(b) + 6e-7f);
    // 1 - k = -expm1(x), x = -p/2
    const float x = -0.5f * p;
    float km1;
    if (x > -0.7f) {
        float q = 1.f / 362880.f;
        q = fmaf(q, x, 1.f / 40320.f);
        q = fmaf(q, x, 1.f / 5040.f);
        q = fmaf(q, x, 1.f / 720.f);
        q = fmaf(q, x, 1.f / 120.f);
        q = fmaf(q, x, 1.f / 24.f);
        q = fmaf(q, x, 1.f / 6.f);
        q = fmaf(q, x, 0.5f);
        q = fmaf(q, x, 1.f);
        km1 = -x * q;
    } else {
        km1 = 1.f - k;
    }
    c.oma = fmaf(o, km1, om);
    const float relp = p > 0.f ? dp / p : 0.f;
    c.eps_oma = 2.f * (relp + 3.6e-7f);
    return c;
}

}  // namespace nx
