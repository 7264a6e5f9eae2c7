// Parity hook for the table-driven fp64 exp / log (nx_fastmath.cuh): evaluates them
// (or CUDA's library routines, for comparison) on caller-given arguments.
#include "nx_fastmath.cuh"
#include "nx_internal.cuh"

namespace nx {
namespace {

__global__ void fastmath_kernel(int fn, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
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
    if (fn < NX_FM_LOG || fn > NX_FM_CUDA_EXP || n < 0 || (n && (!x || !y))) return NX_INVALID_ARGUMENT;
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
