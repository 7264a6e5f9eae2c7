// Parity hook for the table-driven fp64 exp / log (nx_fastmath.cuh): evaluates them
// (or CUDA's library routines, for comparison) on caller-given arguments.
#include "nx_fastmath.cuh"
#include "nx_internal.cuh"

namespace nx {
namespace {

__global__ void fastmath_kernel(int fn, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (fn == NX_FM_CERT) {  // (u, v, gx, gy, o) -> (alpha32, eps, oma32, eps_oma, alpha64)
            if (5 * i + 4 >= n) continue;
            const double* in = x + 5 * i;
            const double u = in[0], v = in[1], gx = in[2], gy = in[3], o = in[4];
            const CertAlpha c = cert_alpha(static_cast<float>(u), static_cast<float>(v), static_cast<float>(2.0 * gx),
                                           static_cast<float>(2.0 * gy), static_cast<float>(o),
                                           static_cast<float>(1.0 - o));
            double lu, lv;
            const double q = fm_axis_power(u, gx, lu) + fm_axis_power(v, gy, lv);
            double* out = y + 5 * i;
            out[0] = c.alpha;
            out[1] = c.eps;
            out[2] = c.oma;
            out[3] = c.eps_oma;
            out[4] = isinf(q) ? 0.0 : o * fm_exp(-0.5 * q);
            continue;
        }
        const double v = x[i];
        double r;
        switch (fn) {
            case NX_FM_LOG: r = fm_log(v); break;
            case NX_FM_EXP: r = fm_exp(v); break;
            case NX_FM_CUDA_LOG: r = log(v); break;
            default: r = exp(v); break;
        }
        y[i] = r;
    }
}

}  // namespace
}  // namespace nx

extern "C" int nx_debug_fastmath(int fn, const double* x, double* y, int64_t n) {
    if (fn < NX_FM_LOG || fn > NX_FM_CERT || n < 0 || (n && (!x || !y))) return NX_INVALID_ARGUMENT;
    if (n == 0) return NX_OK;
    double *dx = nullptr, *dy = nullptr;
    const size_t bytes = static_cast<size_t>(n) * sizeof(double);
    cudaError_t e = cudaMalloc(&dx, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&dy, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        nx::count_launch();
        nx::fastmath_kernel<<<1184, 256>>>(fn, dx, dy, n);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(y, dy, bytes, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    return e == cudaSuccess ? NX_OK : NX_CUDA_ERROR;
}
