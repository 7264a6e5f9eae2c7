// Device -> pinned-host copy kernel for nx_frame_download.
//
// cudaMemcpyAsync D2H streams the frame (191 MB at config 2) through the L2 and
// evicts what the next frame's render keeps there (hash-table levels, composite
// records): measured, a concurrent memcpy slows the render by ~1/3. This kernel
// reads the frame with evict-first (cache-streaming) loads and writes straight into
// the mapped pinned host buffers over PCIe, a few CTAs wide, so the copy overlaps
// the render without displacing its working set. Four 512-thread CTAs keep PCIe
// saturated (3.6 ms for 191 MB) while taking the fewest SM slots from the render
// (measured at config 2: 32 CTAs 4.6 ms, 4 CTAs 4.4 ms per rendered+downloaded frame).
#include <cstdlib>

#include "nx_internal.cuh"

namespace nx {

namespace {

constexpr int kCopyThreads = 512;
constexpr int kUnroll = 4;

__global__ void __launch_bounds__(kCopyThreads) stream_copy_kernel(const CopyJobs jobs) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int k = 0; k < jobs.n; ++k) {
        const uint8_t* src = jobs.j[k].src;
        uint8_t* dst = jobs.j[k].dst;
        const int64_t bytes = static_cast<int64_t>(jobs.j[k].bytes);
        int64_t done = 0;
        if (jobs.j[k].narrow) {  // fp64 -> fp32, two values per thread (16 B read, 8 B written)
            const double* s8 = reinterpret_cast<const double*>(src);
            float* d4 = reinterpret_cast<float*>(dst);
            const int64_t nv = bytes / 8;
            if (((reinterpret_cast<uintptr_t>(src) & 15) | (reinterpret_cast<uintptr_t>(dst) & 7)) == 0) {
                const int64_t n2 = nv / 2;
                const double2* s2 = reinterpret_cast<const double2*>(s8);
                float2* d2 = reinterpret_cast<float2*>(d4);
                for (int64_t i = tid; i < n2; i += nthreads) {
                    const double2 v = __ldcs(s2 + i);
                    __stcs(d2 + i, make_float2(static_cast<float>(v.x), static_cast<float>(v.y)));
                }
                done = n2 * 2;
            }
            for (int64_t i = done + tid; i < nv; i += nthreads) d4[i] = static_cast<float>(s8[i]);
            continue;
        }
        if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
            const int64_t n16 = bytes / 16;
            const int4* s4 = reinterpret_cast<const int4*>(src);
            int4* d4 = reinterpret_cast<int4*>(dst);
            int64_t i = tid;
            for (; i + (kUnroll - 1) * nthreads < n16; i += kUnroll * nthreads) {
                int4 v[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) v[u] = __ldcs(s4 + i + u * nthreads);
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) __stcs(d4 + i + u * nthreads, v[u]);
            }
            for (; i < n16; i += nthreads) __stcs(d4 + i, __ldcs(s4 + i));
            done = n16 * 16;
        }
        for (int64_t b = done + tid; b < bytes; b += nthreads) dst[b] = src[b];
    }
}

}  // namespace

void launch_stream_copy(const CopyJobs& jobs, cudaStream_t s) {
    if (jobs.n == 0) return;
    static const int ctas = [] {
        const char* e = std::getenv("NX_COPY_CTAS");
        const int v = e ? std::atoi(e) : 4;  // measured: 4 CTAs keep PCIe busy with the least interference
        return v < 1 ? 1 : v;
    }();
    count_launch();
    stream_copy_kernel<<<ctas, kCopyThreads, 0, s>>>(jobs);
}

}  // namespace nx
