// Device scan and stable LSD radix sort (hand-written; no CUB).
//
// The render path needs two sorts per frame:
//   1. the global front-to-back order: 64-bit orderable depth keys, values =
//      primitive ids, stable over an id-ascending input => (depth, id) order
//      exactly as std::sort with the reference comparator (renderer.cpp:102-105);
//   2. the per-tile bucketing: tile-id keys over entries emitted in that order,
//      stable => each tile's list is front to back (renderer.cpp:106-110).
// Both are LSD radix sorts with 8-bit digits: per pass a block histogram, an
// exclusive scan over the [digit][block] matrix, and a stable scatter that ranks
// equal digits with warp match + a cross-warp prefix in shared memory.
#include "nx_sort.cuh"

namespace nx {

namespace {

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread (blockDim = kScanThreads).
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int inc = warp_incl_scan(v);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int w = lane < nw ? s_warp[lane] : 0;
        const int wi = warp_incl_scan(w);
        if (lane < nw) s_warp[lane] = wi - w;
        if (lane == nw - 1) s_warp[32] = wi;
    }
    __syncthreads();
    const int r = s_warp[warp] + inc - v;
    if (total) *total = s_warp[32];
    return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int32_t* in, int64_t n,
                                                                   int32_t* block_sums) {
    __shared__ int s_warp[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) v += in[base + k];
    int total;
    block_excl_scan(v, s_warp, &total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Scans up to kScanTile values in one block (exclusive), optional total.
__global__ void __launch_bounds__(kScanThreads) scan_single_kernel(const int32_t* in, int32_t* out,
                                                                   int64_t n, int32_t* total_out,
                                                                   const int32_t* block_offsets) {
    __shared__ int s_warp[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int vals[kScanItems];
    int v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        vals[k] = base + k < n ? in[base + k] : 0;
        v += vals[k];
    }
    int total;
    int run = block_excl_scan(v, s_warp, &total);
    if (block_offsets) run += block_offsets[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += vals[k];
    }
    if (total_out && threadIdx.x == 0 && !block_offsets) *total_out = total;
    if (total_out && block_offsets && blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1)
        *total_out = run;
}

// One block scans n <= kScanLoopMax values in rounds of kScanTile with a carry
// (one launch instead of three for the radix histogram matrices).
__global__ void __launch_bounds__(kScanThreads) scan_loop_kernel(const int32_t* in, int32_t* out, int64_t n,
                                                                 int32_t* total_out) {
    __shared__ int s_warp[33];
    int carry = 0;
    for (int64_t round = 0; round * kScanTile < n; ++round) {
        const int64_t base = round * kScanTile + threadIdx.x * kScanItems;
        int vals[kScanItems];
        int v = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            vals[k] = base + k < n ? in[base + k] : 0;
            v += vals[k];
        }
        int total;
        int run = block_excl_scan(v, s_warp, &total) + carry;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < n) out[base + k] = run;
            run += vals[k];
        }
        carry += total;
        __syncthreads();
    }
    if (total_out && threadIdx.x == 0) *total_out = carry;
}

// n = device count (capped by the host capacity n_cap) when n_dev != nullptr.
__device__ __forceinline__ int64_t dev_count(int64_t n_cap, const int32_t* n_dev) {
    return n_dev ? min(n_cap, static_cast<int64_t>(*n_dev)) : n_cap;
}

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const K* keys, int64_t n_cap,
                                                                   const int32_t* n_dev, int shift,
                                                                   int32_t* hist, int n_blocks) {
    __shared__ int s_hist[kRadixBuckets];
    const int64_t n = dev_count(n_cap, n_dev);
    s_hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRadixTile;
    for (int i = threadIdx.x; i < kRadixTile; i += kRadixThreads) {
        const int64_t g = base + i;
        if (g < n) atomicAdd(&s_hist[static_cast<int>((keys[g] >> shift) & (kRadixBuckets - 1))], 1);
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * n_blocks + blockIdx.x] = s_hist[threadIdx.x];
}

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(const K* __restrict__ keys_in,
                                                                      const uint32_t* __restrict__ vals_in,
                                                                      K* __restrict__ keys_out,
                                                                      uint32_t* __restrict__ vals_out,
                                                                      int64_t n_cap,
                                                                      const int32_t* __restrict__ n_dev,
                                                                      int shift,
                                                                      const int32_t* __restrict__ offsets,
                                                                      int n_blocks) {
    constexpr int kWarps = kRadixThreads / 32;
    __shared__ int s_base[kRadixBuckets];
    __shared__ int s_cnt[kWarps][kRadixBuckets];
    const int64_t n = dev_count(n_cap, n_dev);
    if (static_cast<int64_t>(blockIdx.x) * kRadixTile >= n) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    s_base[tid] = offsets[static_cast<int64_t>(tid) * n_blocks + blockIdx.x];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRadixTile;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int round = 0; round < kRadixTile / kRadixThreads; ++round) {
        const int64_t i = base + static_cast<int64_t>(round) * kRadixThreads + tid;
        if (base + static_cast<int64_t>(round) * kRadixThreads >= n) break;  // uniform
        const bool valid = i < n;
        K k = 0;
        uint32_t v = 0;
        unsigned d = 0xffffffffu;
        if (valid) {
            k = keys_in[i];
            v = vals_in[i];
            d = static_cast<unsigned>((k >> shift) & (kRadixBuckets - 1));
        }
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_cnt[w][tid] = 0;
        __syncthreads();
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt_mask);
        if (valid && rank == 0) s_cnt[warp][d] = __popc(peers);
        __syncthreads();
        int run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = s_cnt[w][tid];
            s_cnt[w][tid] = s_base[tid] + run;
            run += c;
        }
        s_base[tid] += run;
        __syncthreads();
        if (valid) {
            const int pos = s_cnt[warp][d] + rank;
            keys_out[pos] = k;
            vals_out[pos] = v;
        }
        __syncthreads();
    }
}

template <typename K>
bool radix_sort_impl(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n,
                     const int32_t* n_dev, int begin_bit, int end_bit, int32_t* scratch, cudaStream_t stream) {
    if (n <= 1) return false;
    const int n_blocks = static_cast<int>((n + kRadixTile - 1) / kRadixTile);
    const int64_t hist_n = static_cast<int64_t>(n_blocks) * kRadixBuckets;
    int32_t* hist = scratch;
    int32_t* scan_scratch = scratch + hist_n;
    bool in_alt = false;
    for (int bit = begin_bit; bit < end_bit; bit += kRadixBits) {
        K* ki = in_alt ? keys_alt : keys;
        uint32_t* vi = in_alt ? vals_alt : vals;
        K* ko = in_alt ? keys : keys_alt;
        uint32_t* vo = in_alt ? vals : vals_alt;
        count_launch(2);
        radix_hist_kernel<K><<<n_blocks, kRadixThreads, 0, stream>>>(ki, n, n_dev, bit, hist, n_blocks);
        scan_exclusive(hist, hist, hist_n, nullptr, scan_scratch, stream);
        radix_scatter_kernel<K><<<n_blocks, kRadixThreads, 0, stream>>>(ki, vi, ko, vo, n, n_dev, bit, hist,
                                                                        n_blocks);
        in_alt = !in_alt;
    }
    return in_alt;
}

}  // namespace

size_t scan_scratch_ints(int64_t n) {
    const int64_t n_blocks = (n + kScanTile - 1) / kScanTile;
    return static_cast<size_t>(n_blocks) + (n_blocks > 1 ? scan_scratch_ints(n_blocks) : 0) + 8;
}

void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* total, int32_t* scratch,
                    cudaStream_t stream) {
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(int32_t), stream);
        return;
    }
    const int64_t n_blocks = (n + kScanTile - 1) / kScanTile;
    if (n_blocks == 1) {
        count_launch(1);
        scan_single_kernel<<<1, kScanThreads, 0, stream>>>(in, out, n, total, nullptr);
        return;
    }
    if (n <= kScanLoopMax) {
        count_launch(1);
        scan_loop_kernel<<<1, kScanThreads, 0, stream>>>(in, out, n, total);
        return;
    }
    // reduce per block, scan the block sums (recursively), then scan each block with its offset
    count_launch(2);
    scan_reduce_kernel<<<static_cast<unsigned>(n_blocks), kScanThreads, 0, stream>>>(in, n, scratch);
    scan_exclusive(scratch, scratch, n_blocks, nullptr, scratch + n_blocks, stream);
    scan_single_kernel<<<static_cast<unsigned>(n_blocks), kScanThreads, 0, stream>>>(in, out, n, total,
                                                                                    scratch);
}

size_t radix_scratch_ints(int64_t n) {
    const int64_t n_blocks = (n + kRadixTile - 1) / kRadixTile;
    const int64_t hist_n = n_blocks * kRadixBuckets;
    return static_cast<size_t>(hist_n) + scan_scratch_ints(hist_n);
}

bool radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, const int32_t* n_dev, int begin_bit, int end_bit, int32_t* scratch,
                          cudaStream_t stream) {
    return radix_sort_impl<uint64_t>(keys, vals, keys_alt, vals_alt, n, n_dev, begin_bit, end_bit, scratch, stream);
}

bool radix_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                          int64_t n, const int32_t* n_dev, int begin_bit, int end_bit, int32_t* scratch,
                          cudaStream_t stream) {
    return radix_sort_impl<uint32_t>(keys, vals, keys_alt, vals_alt, n, n_dev, begin_bit, end_bit, scratch, stream);
}

}  // namespace nx
