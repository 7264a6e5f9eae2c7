// Device helpers shared by the forward (nx_composite.cu) and backward
// (nx_backward.cu) compositing kernels: the degree-3 SH basis and colour in fp32
// (colour only — no decision depends on it) and the conservative fp32 prefilter.
#pragma once

#include "nx_internal.cuh"

namespace nx {

// sh_basis (sh.hpp:11-40), 3DGS sign convention, fp32.
__device__ __forceinline__ void sh_basis_f32(float x, float y, float z, float* b) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[0] = 0.28209479177387814f;
    b[1] = -0.4886025119029199f * y;
    b[2] = 0.4886025119029199f * z;
    b[3] = -0.4886025119029199f * x;
    b[4] = 1.0925484305920792f * x * y;
    b[5] = -1.0925484305920792f * y * z;
    b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    b[7] = -1.0925484305920792f * x * z;
    b[8] = 0.5462742152960396f * (xx - yy);
    b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    b[10] = 2.890611442640554f * x * y * z;
    b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// Primitive SH colour (eval_sh / eval_sh_cached, sh.hpp:46-73) in fp32 from the ray
// direction. `active` (optional) receives the clamp mask bit c = (acc_c >= 0), the
// mask eval_sh_backward uses (sh.hpp:76-83).
__device__ __forceinline__ void eval_sh_f32(const float* __restrict__ sh, float x, float y, float z, int degree,
                                            float* rgb, uint32_t* active = nullptr) {
    float a0 = 0.5f + 0.28209479177387814f * __ldg(sh + 0);
    float a1 = 0.5f + 0.28209479177387814f * __ldg(sh + 1);
    float a2 = 0.5f + 0.28209479177387814f * __ldg(sh + 2);
    if (degree >= 3) {
        float b[16];
        sh_basis_f32(x, y, z, b);
        const float4* s4 = reinterpret_cast<const float4*>(sh);
        float c[48];
#pragma unroll
        for (int q = 0; q < 12; ++q) {
            const float4 v = __ldg(s4 + q);
            c[4 * q + 0] = v.x;
            c[4 * q + 1] = v.y;
            c[4 * q + 2] = v.z;
            c[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int k = 1; k < 16; ++k) {
            a0 = fmaf(c[3 * k + 0], b[k], a0);
            a1 = fmaf(c[3 * k + 1], b[k], a1);
            a2 = fmaf(c[3 * k + 2], b[k], a2);
        }
    }
    if (active) *active = (a0 >= 0.f ? 1u : 0u) | (a1 >= 0.f ? 2u : 0u) | (a2 >= 0.f ? 4u : 0u);
    rgb[0] = fmaxf(a0, 0.f);
    rgb[1] = fmaxf(a1, 0.f);
    rgb[2] = fmaxf(a2, 0.f);
}

// sh_basis + eval_sh (sh.hpp:11-57) in fp64, the reference's operation order
// (acc = 0.5, then acc += coeff_k * basis_k for k = 0, 1, ...): the NX_PRECISION_F64 colour.
__device__ __forceinline__ void eval_sh_f64(const double* sh, const double* d, int degree, double* rgb) {
    double b[16];
    const double x = d[0], y = d[1], z = d[2];
    const double xx = x * x, yy = y * y, zz = z * z;
    b[0] = 0.28209479177387814;
    b[1] = -0.4886025119029199 * y;
    b[2] = 0.4886025119029199 * z;
    b[3] = -0.4886025119029199 * x;
    b[4] = 1.0925484305920792 * x * y;
    b[5] = -1.0925484305920792 * y * z;
    b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    b[7] = -1.0925484305920792 * x * z;
    b[8] = 0.5462742152960396 * (xx - yy);
    b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    b[10] = 2.890611442640554 * x * y * z;
    b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    b[14] = 1.445305721320277 * z * (xx - yy);
    b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
    const int n = degree >= 3 ? 16 : 1;
    for (int c = 0; c < 3; ++c) {
        double acc = 0.5;
        for (int k = 0; k < n; ++k) acc += sh[k * 3 + c] * b[k];
        rgb[c] = acc < 0.0 ? 0.0 : acc;
    }
}

// fp32 conservative prefilter: false only if the exact test provably misses
// (t <= near_eps, or |u| > ru, or |v| > rv).
__device__ __forceinline__ bool prefilter(const float4* f, float dfx, float dfy, float dfz, float near_eps_f) {
    const float4 f0 = f[0];
    const float denom = dfx * f0.x + dfy * f0.y + dfz * f0.z;
    if (!(fabsf(denom) >= 1e-2f)) return true;  // grazing: leave it to the exact path
    const float ta = __fdividef(f0.w, denom);
    if (!(ta * (1.0f + 1e-4f) > near_eps_f)) return false;  // t <= near_eps for sure
    const float4 f1 = f[1], f2 = f[2], f3 = f[3];
    const float ta1 = ta * (dfx * f1.x + dfy * f1.y + dfz * f1.z);
    const float du = ta1 - f1.w;
    if (fabsf(du) > f3.x + (1e-4f * (fabsf(ta1) + fabsf(ta) + fabsf(f1.w)) + 1e-7f)) return false;
    const float ta2 = ta * (dfx * f2.x + dfy * f2.y + dfz * f2.z);
    const float dv = ta2 - f2.w;
    return !(fabsf(dv) > f3.y + (1e-4f * (fabsf(ta2) + fabsf(ta) + fabsf(f2.w)) + 1e-7f));
}

}  // namespace nx
