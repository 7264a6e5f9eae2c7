// fp64 peak microbenchmark (B200): independent DFMA chains on every SM, timed with
// CUDA events. The compositing kernel's fp64 roofline in bench.py is stated against
// this measured number (MEASURED_PEAKS.json has HBM and bf16 only).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp64_peak tools/fp64_peak.cu
//   build/fp64_peak > profiles/r02/fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-9);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * kChains * kIters * double(blocks) * threads;
    const double tf = flops / (best * 1e-3) / 1e12;
    const double per_clk_sm = flops / 2.0 / (best * 1e-3) / (sms * clk * 1e3);
    std::printf("{\"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm\": %.2f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
                "\"best_ms\": %.4f, \"how\": \"%d CTAs x %d threads, %d independent DFMA chains x %d iterations, "
                "best of 10 (CUDA events); 2 flops per DFMA\"}\n",
                tf, per_clk_sm, sms, clk / 1e3, best, blocks, threads, kChains, kIters);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
