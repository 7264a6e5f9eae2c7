// Device scan and stable LSD radix sort (hand-written; no CUB).
//
// The render path needs two sorts per frame:
//   1. the global front-to-back order: 64-bit orderable depth keys, values =
//      primitive ids, stable over an id-ascending input => (depth, id) order
//      exactly as std::sort with the reference comparator (renderer.cpp:102-105);
//   2. the per-tile bucketing: tile-id keys over entries emitted in that order,
//      stable => each tile's list is front to back (renderer.cpp:106-110).
// Both are one-sweep LSD radix sorts with 8-bit digits: one upsweep launch builds the
// global digit histograms of every pass; then one launch per pass ranks its block of
// keys stably (warp match + cross-warp prefix in shared memory), publishes the block's
// digit counts and finds its digit offsets by decoupled look-back over the preceding
// blocks, then scatters. A pass whose keys all share one digit is a plain copy.
// The exclusive scan is single-pass with the same look-back. Blocks take their index
// from an atomic ticket (in launch order), so every block they wait on is running.
// Counts may live on the device (n_dev): grids are sized by the host capacity and the
// blocks past the device count leave at once (no host round trip).
#include "nx_sort.cuh"
#include "../../include/nexel_b200.h"

#include <algorithm>

namespace nx {

namespace {

constexpr uint32_t kFlagAgg = 1u, kFlagIncl = 2u;  // look-back status: aggregate / inclusive prefix

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread.
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
    __syncthreads();
    return r;
}

__device__ __forceinline__ void st_status(uint64_t* p, uint32_t flag, uint32_t v) {
    const unsigned long long w = (static_cast<unsigned long long>(flag) << 32) | v;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// Exclusive prefix of `agg` over the blocks before `b` by decoupled look-back on
// status[0..b) (stride `stride` between consecutive blocks' words). One thread. The
// words of kLookBatch predecessors are loaded together (independent loads in flight),
// then consumed in order: a chain of b aggregates costs ~b / kLookBatch L2 round trips
// instead of b (all blocks publish their aggregates at about the same time, so without
// the batch the last block walks the whole chain one dependent load at a time).
#ifndef NX_LOOK_BATCH
#define NX_LOOK_BATCH 8
#endif
constexpr int kLookBatch = NX_LOOK_BATCH;
__device__ __forceinline__ uint32_t look_back(const uint64_t* status, int64_t stride, int b) {
    uint32_t run = 0;
    int p = b - 1;
    while (p >= 0) {
        uint64_t w[kLookBatch];
#pragma unroll
        for (int i = 0; i < kLookBatch; ++i) w[i] = p - i >= 0 ? ld_status(status + (p - i) * stride) : 0ull;
        int used = 0;
        bool done = false;
#pragma unroll
        for (int i = 0; i < kLookBatch; ++i) {
            if (done || used < i) continue;  // stopped at an earlier word
            if (p - i < 0) {
                done = true;
                continue;
            }
            const uint32_t flag = static_cast<uint32_t>(w[i] >> 32);
            if (flag == 0) continue;  // not published yet (it is running: ticket order): reload from here
            run += static_cast<uint32_t>(w[i]);
            used = i + 1;
            if (flag == kFlagIncl) done = true;
        }
        if (done) break;
        p -= used;
    }
    return run;
}

// n = device count (capped by the host capacity n_cap) when n_dev != nullptr.
__device__ __forceinline__ int64_t dev_count(int64_t n_cap, const int32_t* n_dev) {
    return n_dev ? min(n_cap, static_cast<int64_t>(max(*n_dev, 0))) : n_cap;
}

// ---------------------------------------------------------------- single-pass scan
// scratch: [0] ticket, [2..] status words (64-bit) per block
__global__ void __launch_bounds__(kScanThreads) scan_onepass_kernel(const int32_t* in, int32_t* out, int64_t n,
                                                                    int32_t* total_out, int32_t* scratch) {
    __shared__ int s_warp[33];
    __shared__ int s_block, s_prefix;
    uint64_t* status = reinterpret_cast<uint64_t*>(scratch + 2);
    if (threadIdx.x == 0) s_block = atomicAdd(scratch, 1);
    __syncthreads();
    const int b = s_block;
    const int64_t base = static_cast<int64_t>(b) * kScanTile + threadIdx.x * kScanItems;
    int vals[kScanItems];
    int v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        vals[k] = base + k < n ? in[base + k] : 0;
        v += vals[k];
    }
    int total;
    int run = block_excl_scan(v, s_warp, &total);
    if (threadIdx.x == 0) {
        if (b == 0) {
            st_status(status, kFlagIncl, static_cast<uint32_t>(total));
            s_prefix = 0;
        } else {
            st_status(status + b, kFlagAgg, static_cast<uint32_t>(total));
            const uint32_t pre = look_back(status, 1, b);
            st_status(status + b, kFlagIncl, pre + static_cast<uint32_t>(total));
            s_prefix = static_cast<int>(pre);
        }
    }
    __syncthreads();
    run += s_prefix;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += vals[k];
    }
    if (total_out && b == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) *total_out = run;
}

// ---------------------------------------------------------------- one-sweep radix sort
// scratch layout (int32 units): [0..16) tickets per pass, [16..16+256*8) global digit
// histograms of up to 8 passes, then status words: pass p, block b, digit d at
// status[(p * n_blocks + b) * 256 + d].
constexpr int kMaxPasses = 8;
constexpr int kHistOff = 16;
constexpr int kStatusOff = kHistOff + kMaxPasses * kRadixBuckets;  // even: 64-bit aligned
template <typename K>
constexpr int tile_of() {  // keys per block per pass
    return sizeof(K) == 8 ? kRadixTile64 : kRadixTile;
}
static_assert(kRadixTile % kRadixThreads == 0 && kRadixTile64 % kRadixThreads == 0, "whole items per thread");

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) radix_upsweep_kernel(const K* keys, int64_t n_cap,
                                                                      const int32_t* n_dev, int begin_bit,
                                                                      int passes, int32_t* hist) {
    __shared__ int s_hist[kMaxPasses][kRadixBuckets];
    const int64_t n = dev_count(n_cap, n_dev);
    for (int p = 0; p < passes; ++p) s_hist[p][threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const K k = keys[i];
        for (int p = 0; p < passes; ++p)
            atomicAdd(&s_hist[p][static_cast<int>((k >> (begin_bit + p * kRadixBits)) & (kRadixBuckets - 1))], 1);
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
        if (s_hist[p][threadIdx.x]) atomicAdd(&hist[p * kRadixBuckets + threadIdx.x], s_hist[p][threadIdx.x]);
}

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) radix_pass_kernel(const K* __restrict__ keys_in,
                                                                   const uint32_t* __restrict__ vals_in,
                                                                   K* __restrict__ keys_out,
                                                                   uint32_t* __restrict__ vals_out, int64_t n_cap,
                                                                   const int32_t* __restrict__ n_dev, int shift,
                                                                   int pass, int n_blocks, int32_t* scratch) {
    constexpr int kWarps = kRadixThreads / 32;
    constexpr int kTile = tile_of<K>();
    constexpr int kRadixItems = kTile / kRadixThreads;  // per thread
    __shared__ int s_cnt[kWarps][kRadixBuckets];
    __shared__ int s_local[kRadixBuckets];  // block-local running count per digit
    __shared__ int s_glob[kRadixBuckets];   // global base of each digit for this block
    __shared__ int s_warp[33];
    __shared__ int s_block, s_trivial;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = dev_count(n_cap, n_dev);
    if (tid == 0) s_block = atomicAdd(scratch + pass, 1);
    const int hcount = scratch[kHistOff + pass * kRadixBuckets + tid];
    if (tid == 0) s_trivial = 0;
    __syncthreads();
    if (hcount == n) s_trivial = 1;  // every key has this digit: the pass is a copy
    const int b = s_block;
    const int64_t base = static_cast<int64_t>(b) * kTile;
    __syncthreads();
    if (base >= n) return;
    if (s_trivial) {
        for (int i = tid; i < kTile; i += kRadixThreads)
            if (base + i < n) {
                keys_out[base + i] = keys_in[base + i];
                vals_out[base + i] = vals_in[base + i];
            }
        return;
    }
    // exclusive scan of the pass's global histogram: the digit's start in the output
    const int gstart = block_excl_scan(hcount, s_warp, nullptr);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_cnt[w][tid] = 0;
    __syncthreads();
    // Warp w ranks the tile's w-th run of 32 * kRadixItems keys (index order = warp, item,
    // lane): per-warp digit counts in shared memory, peers found with match_any, only
    // warp-level synchronisation until the per-digit offsets over the warps.
    const unsigned lt_mask = (1u << lane) - 1u;
    K key[kRadixItems];
    uint32_t val[kRadixItems];
    int loc[kRadixItems];
    unsigned dig[kRadixItems];
    const int64_t wbase = base + static_cast<int64_t>(warp) * (32 * kRadixItems);
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? keys_in[i] : K(0);
        val[r] = valid ? vals_in[i] : 0u;
        dig[r] = valid ? static_cast<unsigned>((key[r] >> shift) & (kRadixBuckets - 1)) : 0xffffffffu;
    }
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        const unsigned peers = __match_any_sync(0xffffffffu, dig[r]);
        const int rank = __popc(peers & lt_mask);
        const bool valid = dig[r] != 0xffffffffu;
        const int pre = valid ? s_cnt[warp][dig[r]] : 0;
        __syncwarp();
        if (valid && rank == 0) s_cnt[warp][dig[r]] = pre + __popc(peers);
        __syncwarp();
        loc[r] = pre + rank;
    }
    __syncthreads();
    {  // digit tid: the warps' exclusive offsets inside the tile and the tile's count
        int run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = s_cnt[w][tid];
            s_cnt[w][tid] = run;
            run += c;
        }
        s_local[tid] = run;
    }
    // publish this block's digit counts, look back for the preceding blocks' totals
    uint64_t* status = reinterpret_cast<uint64_t*>(scratch + kStatusOff) +
                       static_cast<int64_t>(pass) * n_blocks * kRadixBuckets;
    const uint32_t mine = static_cast<uint32_t>(s_local[tid]);
    if (b == 0) {
        st_status(status + tid, kFlagIncl, mine);
        s_glob[tid] = gstart;
    } else {
        st_status(status + static_cast<int64_t>(b) * kRadixBuckets + tid, kFlagAgg, mine);
        const uint32_t pre = look_back(status + tid, kRadixBuckets, b);
        st_status(status + static_cast<int64_t>(b) * kRadixBuckets + tid, kFlagIncl, pre + mine);
        s_glob[tid] = gstart + static_cast<int>(pre);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
        if (dig[r] == 0xffffffffu) continue;
        const int pos = s_glob[dig[r]] + s_cnt[warp][dig[r]] + loc[r];
        keys_out[pos] = key[r];
        vals_out[pos] = val[r];
    }
}

template <typename K>
bool radix_sort_impl(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, int64_t n, const int32_t* n_dev,
                     int begin_bit, int end_bit, int32_t* scratch, cudaStream_t stream) {
    if (n <= 1) return false;
    const int n_blocks = static_cast<int>((n + tile_of<K>() - 1) / tile_of<K>());
    const int passes = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
    if (passes <= 0) return false;
    // tickets + histograms + status words start at zero
    cudaMemsetAsync(scratch, 0,
                    (kStatusOff + static_cast<size_t>(2) * passes * n_blocks * kRadixBuckets) * sizeof(int32_t),
                    stream);
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int up_grid = static_cast<int>(std::min<int64_t>((n + kRadixThreads - 1) / kRadixThreads, 4 * sms));
    count_launch(1 + passes);
    radix_upsweep_kernel<K><<<up_grid, kRadixThreads, 0, stream>>>(keys, n, n_dev, begin_bit, passes,
                                                                     scratch + kHistOff);
    bool in_alt = false;
    for (int p = 0; p < passes; ++p) {
        K* ki = in_alt ? keys_alt : keys;
        uint32_t* vi = in_alt ? vals_alt : vals;
        K* ko = in_alt ? keys : keys_alt;
        uint32_t* vo = in_alt ? vals : vals_alt;
        radix_pass_kernel<K><<<n_blocks, kRadixThreads, 0, stream>>>(ki, vi, ko, vo, n, n_dev,
                                                                     begin_bit + p * kRadixBits, p, n_blocks, scratch);
        in_alt = !in_alt;
    }
    return in_alt;
}

}  // namespace

size_t scan_scratch_ints(int64_t n) {
    const int64_t n_blocks = (n + kScanTile - 1) / kScanTile;
    return static_cast<size_t>(2 + 2 * n_blocks + 8);
}

void scan_exclusive(const int32_t* in, int32_t* out, int64_t n, int32_t* total, int32_t* scratch,
                    cudaStream_t stream) {
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(int32_t), stream);
        return;
    }
    const int64_t n_blocks = (n + kScanTile - 1) / kScanTile;
    cudaMemsetAsync(scratch, 0, (2 + 2 * n_blocks) * sizeof(int32_t), stream);
    count_launch(1);
    scan_onepass_kernel<<<static_cast<unsigned>(n_blocks), kScanThreads, 0, stream>>>(in, out, n, total, scratch);
}

size_t radix_scratch_ints(int64_t n) {
    const int64_t n_blocks = (n + kRadixTile - 1) / kRadixTile;
    return static_cast<size_t>(kStatusOff + 2 * kMaxPasses * n_blocks * kRadixBuckets + 8);
}

size_t radix_scratch_ints64(int64_t n) {
    const int64_t n_blocks = (n + kRadixTile64 - 1) / kRadixTile64;
    return static_cast<size_t>(kStatusOff + 2 * kMaxPasses * n_blocks * kRadixBuckets + 8);
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

// ---------------------------------------------------------------- parity entry points
extern "C" int nx_debug_radix_sort(int key_bytes, void* keys, uint32_t* vals, int64_t n, int64_t cap, int begin_bit,
                                   int end_bit) {
    if ((key_bytes != 4 && key_bytes != 8) || n < 0 || cap < n || begin_bit < 0 || end_bit > 8 * key_bytes ||
        begin_bit > end_bit || (n && (!keys || !vals)) || n > INT32_MAX)
        return NX_INVALID_ARGUMENT;
    if (n == 0) return NX_OK;
    const size_t kb = static_cast<size_t>(cap) * key_bytes, vb = static_cast<size_t>(cap) * sizeof(uint32_t);
    uint8_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr;
    int32_t* sc = nullptr;
    cudaError_t e = cudaMalloc(&k0, kb);
    if (e == cudaSuccess) e = cudaMalloc(&k1, kb);
    if (e == cudaSuccess) e = cudaMalloc(&v0, vb);
    if (e == cudaSuccess) e = cudaMalloc(&v1, vb);
    const size_t sc_ints = std::max(nx::radix_scratch_ints(cap), nx::radix_scratch_ints64(cap));
    if (e == cudaSuccess) e = cudaMalloc(&sc, (sc_ints + 1) * sizeof(int32_t));
    int32_t* n_dev = sc ? sc + sc_ints : nullptr;
    const int32_t n32 = static_cast<int32_t>(n);
    if (e == cudaSuccess) e = cudaMemset(k0, 0xff, kb);  // past the count: garbage the sort must not read
    if (e == cudaSuccess) e = cudaMemcpy(k0, keys, static_cast<size_t>(n) * key_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(v0, vals, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(n_dev, &n32, sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        bool alt;
        if (key_bytes == 8)
            alt = nx::radix_sort_pairs_u64(reinterpret_cast<uint64_t*>(k0), v0, reinterpret_cast<uint64_t*>(k1), v1,
                                           cap, n_dev, begin_bit, end_bit, sc, nullptr);
        else
            alt = nx::radix_sort_pairs_u32(reinterpret_cast<uint32_t*>(k0), v0, reinterpret_cast<uint32_t*>(k1), v1,
                                           cap, n_dev, begin_bit, end_bit, sc, nullptr);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpy(keys, alt ? k1 : k0, static_cast<size_t>(n) * key_bytes, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(vals, alt ? v1 : v0, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost);
    }
    cudaFree(k0);
    cudaFree(k1);
    cudaFree(v0);
    cudaFree(v1);
    cudaFree(sc);
    return e == cudaSuccess ? NX_OK : NX_CUDA_ERROR;
}

extern "C" int nx_debug_scan(const int32_t* in, int32_t* out, int64_t n, int64_t cap, int32_t* total) {
    if (n < 0 || cap < n || (n && (!in || !out))) return NX_INVALID_ARGUMENT;
    int32_t *d = nullptr, *sc = nullptr;
    const size_t bytes = static_cast<size_t>(cap > 0 ? cap : 1) * sizeof(int32_t);
    cudaError_t e = cudaMalloc(&d, bytes + sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&sc, nx::scan_scratch_ints(cap) * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemset(d, 0, bytes + sizeof(int32_t));
    if (e == cudaSuccess && n) e = cudaMemcpy(d, in, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyHostToDevice);
    int32_t* d_total = d + (cap > 0 ? cap : 1);
    if (e == cudaSuccess) {
        nx::scan_exclusive(d, d, cap, d_total, sc, nullptr);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && n) e = cudaMemcpy(out, d, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && total) e = cudaMemcpy(total, d_total, sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(sc);
    return e == cudaSuccess ? NX_OK : NX_CUDA_ERROR;
}
