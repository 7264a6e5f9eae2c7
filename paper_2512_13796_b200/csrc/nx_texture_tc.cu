// K7 texture, tensor-core variant for the reference field shape (16 levels x 2
// features -> 32 -> 64 -> 64 -> 48): hash-grid gathers on the SIMT pipes, the
// bias-free ReLU MLP (TextureMlp::forward, mlp.cpp:24-43) on the 5th-gen tensor
// cores (tcgen05.mma, accumulators in TMEM), SH colour (eval_sh, sh.hpp:46-57)
// and the Eq. 7 composite (renderer.cpp:219-236) in the epilogue.
//
// Persistent CTAs of 128 threads, three per SM: one tile = 128 top-K slots of an
// 8-pixel-wide block (neighbouring rows query neighbouring lattice cells) = the
// M = 128 rows of every MMA, one thread per row (= its TMEM lane). Per tile:
//   gather   16 levels per row (grid_lookup, hash_grid.cpp:26-83; lattice position,
//            floor and hashing in fp64/int64 like the reference, so the same table
//            rows are read), two-stage software pipeline -> 32 features -> smem
//   layer 1  D = F[128x32] . W1^T          (TMEM cols 0..63)
//   layer 2  D = relu(D) . W2^T            (same columns, drained first)
//   layer 3  D = relu(D) . W3^T  [128x48]
//   epilogue tcgen05.ld -> 48 SH coefficients -> rgb -> texture, final (Eq. 7).
// Three CTAs per SM keep three such pipelines in flight, so one CTA's MMA wait
// overlaps another's gathers. fp32-class accuracy from bf16 operands via the
// 3-term split a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi (relative error ~2^-16),
// accumulated in fp32 in TMEM. Operands use the K-major no-swizzle canonical
// layout: 8-row x 16-byte core matrices, LBO = 128 B (next K chunk),
// SBO = 128*K/8 B (next 8-row group).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "nx_composite.cuh"
#include "nx_grid.cuh"
#include "nx_tc.cuh"

namespace nx {

namespace {

constexpr int kTcThreads = 128;
constexpr int kRows = 128;
constexpr int kIn = 32, kHid = 64, kOut = 48;
// D1, D2 and D3 share columns 0..63: each is drained (tcgen05.ld + wait + fence +
// barrier) before the next layer's MMAs overwrite it.
constexpr uint32_t kTmemCols = 64;

// shared-memory carve-up (bytes)
constexpr int kOffW1h = 0;
constexpr int kOffW1l = kOffW1h + kHid * kIn * 2;    // 4 KB each
constexpr int kOffW2h = kOffW1l + kHid * kIn * 2;
constexpr int kOffW2l = kOffW2h + kHid * kHid * 2;   // 8 KB each
constexpr int kOffW3h = kOffW2l + kHid * kHid * 2;
constexpr int kOffW3l = kOffW3h + kOut * kHid * 2;   // 6 KB each
constexpr int kOffAh = kOffW3l + kOut * kHid * 2;
constexpr int kOffAl = kOffAh + kRows * kHid * 2;    // 16 KB each
constexpr int kOffRgb = kOffAl + kRows * kHid * 2;   // float [128][3]
constexpr int kOffBar = kOffRgb + kRows * 3 * 4;     // mbarrier (8 B)
constexpr int kOffTmem = kOffBar + 8;                // tmem base (4 B)
constexpr int kSmemUsed = kOffTmem + 8;              // ~70.5 KB: three CTAs per SM
static_assert(kSmemUsed <= 72 * 1024, "three CTAs per SM");
constexpr int kCtasPerSm = 3;


// Issues one layer: D = A . B^T over K (3 split terms per 16-wide k-step), commit.
__device__ __forceinline__ void issue_layer(uint8_t* smem, uint32_t dtm, int off_bh, int off_bl, int K,
                                            uint32_t idesc, uint32_t bar) {
    tc_fence_after();
    const uint32_t ah = smem_u32(smem + kOffAh), al = smem_u32(smem + kOffAl);
    const uint32_t bh = smem_u32(smem + off_bh), bl = smem_u32(smem + off_bl);
    const uint32_t sbo = 16 * K;
    for (int s = 0; s < K / 16; ++s) {
        const uint32_t o = s * 256;
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, s > 0);
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bl + o, 128, sbo), idesc, 1);
        mma_bf16(dtm, smem_desc(al + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, 1);
    }
    mma_commit(bar);
}

__global__ void __launch_bounds__(kTcThreads, kCtasPerSm) texture_tc_kernel(const TextureArgs a, const TcConst cst,
                                                                            int bw, int bh, int tiles_x,
                                                                            int64_t n_tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kOffBar);

    // ---- one-time setup: weights -> smem (bf16 hi/lo, K-major core-matrix layout)
    for (int e = tid; e < kHid * kIn / 8; e += kTcThreads) {  // W1 [64][32]
        const int n = e / (kIn / 8), c = e % (kIn / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w1 + n * kIn + c * 8 + i);
        store_split8(smem, kOffW1h, kOffW1l, kmajor_off(n, c * 8, kIn), x);
    }
    for (int e = tid; e < kHid * kHid / 8; e += kTcThreads) {  // W2 [64][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w2 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW2h, kOffW2l, kmajor_off(n, c * 8, kHid), x);
    }
    for (int e = tid; e < kOut * kHid / 8; e += kTcThreads) {  // W3 [48][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w3 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW3h, kOffW3l, kmajor_off(n, c * 8, kHid), x);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kOffTmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kOffTmem);
    uint32_t phase = 0;

    const int K = a.fb.K;
    const int W = a.cam.W;
    const int row = tid;  // MMA row == TMEM lane 32 * warp + lane
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * warp) << 16);
    const uint32_t T = 1u << a.scene.field.log2_table;
    const uint32_t mask = T - 1u;
    const float2* tab = reinterpret_cast<const float2*>(a.scene.table);
    float* srgb = reinterpret_cast<float*>(smem + kOffRgb);
    constexpr uint32_t kIdesc64 = idesc_bf16_f32(kRows, 64);
    constexpr uint32_t kIdesc48 = idesc_bf16_f32(kRows, 48);
    int n_queries = 0;

    const int ppt = bw * bh;  // pixels per tile; rows = ppt * K <= 128
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        // row -> (pixel of the bw x bh block, slot j): neighbouring rows are neighbouring pixels
        const int tpx = static_cast<int>(tile % tiles_x) * bw, tpy = static_cast<int>(tile / tiles_x) * bh;
        const int p_in = row / K, j_in = row - (row / K) * K;
        const int px = tpx + p_in % bw, py = tpy + p_in / bw;
        const bool in_tile = p_in < ppt && px < W && py < a.cam.H;
        const int64_t slot = in_tile ? (static_cast<int64_t>(py) * W + px) * K + j_in : 0;
        const bool valid = in_tile && a.fb.ids[slot] >= 0;
        n_queries += valid;
        double dir[3] = {0.0, 0.0, 1.0};
        float feats[kIn];
        if (valid) {
            pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
            const double t = a.fb.depths[slot];
            const double x0 = a.cam.o[0] + t * dir[0];  // build_queries (renderer.cpp:196-198)
            const double x1 = a.cam.o[1] + t * dir[1];
            const double x2 = a.cam.o[2] + t * dir[2];
            const float ft = static_cast<float>(a.cam.fx / t);
            const bool small = fmax(fabs(x0), fmax(fabs(x1), fabs(x2))) * cst.level_scale[kLevels - 1] < 1073741824.0;
            if (small) {
                // two-stage software pipeline: level l+1's 8 gathers are in flight while
                // level l is interpolated
                LevelFetch cur = fetch_level<true>(0, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
#pragma unroll
                for (int l = 0; l < kLevels; ++l) {
                    LevelFetch nxt;
                    if (l + 1 < kLevels)
                        nxt = fetch_level<true>(l + 1, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
                    const float2 g = interp(cur);
                    feats[2 * l] = g.x;
                    feats[2 * l + 1] = g.y;
                    if (l + 1 < kLevels) cur = nxt;
                }
            } else {  // far-away samples: 64-bit lattice coordinates (rare; not pipelined)
#pragma unroll
                for (int l = 0; l < kLevels; ++l) {
                    const float2 g =
                        interp(fetch_level<false>(l, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight));
                    feats[2 * l] = g.x;
                    feats[2 * l + 1] = g.y;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < kIn; ++i) feats[i] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < kIn / 8; ++c) store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 8 * c, kIn), feats + 8 * c);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();

        // ---- layer 1: D = F . W1^T (K = 32)
        if (tid == 0) issue_layer(smem, tmem, kOffW1h, kOffW1l, kIn, kIdesc64, bar);
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();

        // ---- hidden layers: relu(D) -> A (K = 64), then D = A . W^T
#pragma unroll 1
        for (int layer = 0; layer < 2; ++layer) {
#if NX_TMEM_BATCH
            {
                uint32_t r[kHid];
                tmem_ld_batch<kHid / 16>(taddr, r);
#pragma unroll
                for (int c = 0; c < kHid / 8; ++c) {
                    float v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = fmaxf(__uint_as_float(r[8 * c + i]), 0.f);
                    store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 8 * c, kHid), v);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < kHid / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c, kHid), v);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c + 8, kHid), v + 8);
            }
#endif
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                if (layer == 0) issue_layer(smem, tmem, kOffW2h, kOffW2l, kHid, kIdesc64, bar);
                else issue_layer(smem, tmem, kOffW3h, kOffW3l, kHid, kIdesc48, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            tc_fence_after();
        }

        // ---- epilogue: D (48 SH coefficients, k*3 + c) -> rgb (eval_sh, sh.hpp:46-57)
        {
            const float x = static_cast<float>(dir[0]), y = static_cast<float>(dir[1]), z = static_cast<float>(dir[2]);
            const float xx = x * x, yy = y * y, zz = z * z;
            float b[16];
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
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
            for (int c = 0; c < kOut / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int o = 16 * c + i, k = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v[i], b[k], c0);
                    else if (o % 3 == 1) c1 = fmaf(v[i], b[k], c1);
                    else c2 = fmaf(v[i], b[k], c2);
                }
            }
            float rgb[3] = {0.f, 0.f, 0.f};
            if (valid) {
                rgb[0] = fmaxf(0.5f + c0, 0.f);
                rgb[1] = fmaxf(0.5f + c1, 0.f);
                rgb[2] = fmaxf(0.5f + c2, 0.f);
            }
            srgb[row * 3 + 0] = rgb[0];
            srgb[row * 3 + 1] = rgb[1];
            srgb[row * 3 + 2] = rgb[2];
            if (in_tile) {
                a.fb.texture[slot * 3 + 0] = rgb[0];
                a.fb.texture[slot * 3 + 1] = rgb[1];
                a.fb.texture[slot * 3 + 2] = rgb[2];
            }
        }
        tc_fence_before();
        __syncthreads();
        // ---- Eq. 7: final = base + sum_j W[p,j] * texture[p,j] for this tile's pixels
        if (tid < ppt) {
            const int qx = tpx + tid % bw, qy = tpy + tid / bw;
            if (qx < W && qy < a.cam.H) {
                const int64_t pix = static_cast<int64_t>(qy) * W + qx;
                double acc0 = a.fb.base[pix * 3 + 0], acc1 = a.fb.base[pix * 3 + 1], acc2 = a.fb.base[pix * 3 + 2];
                for (int j = 0; j < K; ++j) {
                    const int64_t sl = pix * K + j;
                    if (a.fb.ids[sl] < 0) continue;
                    const double w = a.fb.weights[sl];
                    const float* tc = srgb + (tid * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
                a.fb.final_img[pix * 3 + 0] = static_cast<float>(acc0);
                a.fb.final_img[pix * 3 + 1] = static_cast<float>(acc1);
                a.fb.final_img[pix * 3 + 2] = static_cast<float>(acc2);
            }
        }
        // srgb and the A buffers are rewritten by the next tile only after its gather,
        // which every thread reaches after this point; the gather's barrier orders them.
    }

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_queries += __shfl_down_sync(0xffffffffu, n_queries, o);
    if ((tid & 31) == 0 && n_queries) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_queries));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------- split variant
// The same pass as two kernels: (1) the hash-grid gathers at full occupancy, one thread
// per slot, features to a per-frame scratch (128 B per slot); (2) the MLP on tcgen05
// over tiles of whole pixels (128/K pixels x K slots), SH colour, texture and Eq. 7.
// The gathers are latency-bound and want many warps; the fused kernel can keep only
// three 128-thread CTAs per SM resident (registers, shared memory).
__global__ void __launch_bounds__(128) tex_features_kernel(const TextureArgs a, const TcConst cst, int64_t total) {
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (sl >= total) return;
    float feats[kIn];
#pragma unroll
    for (int i = 0; i < kIn; ++i) feats[i] = 0.f;
    if (a.fb.ids[sl] >= 0) {
        const int K = a.fb.K;
        const int64_t pix = sl / K;
        double dir[3];
        pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
        const double t = a.fb.depths[sl];
        const double x0 = a.cam.o[0] + t * dir[0], x1 = a.cam.o[1] + t * dir[1], x2 = a.cam.o[2] + t * dir[2];
        const float ft = static_cast<float>(a.cam.fx / t);
        const uint32_t T = 1u << a.scene.field.log2_table, mask = T - 1u;
        const float2* tab = reinterpret_cast<const float2*>(a.scene.table);
        const bool small = fmax(fabs(x0), fmax(fabs(x1), fabs(x2))) * cst.level_scale[kLevels - 1] < 1073741824.0;
        if (small) {
            LevelFetch cur = fetch_level<true>(0, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
#pragma unroll
            for (int l = 0; l < kLevels; ++l) {
                LevelFetch nxt;
                if (l + 1 < kLevels) nxt = fetch_level<true>(l + 1, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
                const float2 g = interp(cur);
                feats[2 * l] = g.x;
                feats[2 * l + 1] = g.y;
                if (l + 1 < kLevels) cur = nxt;
            }
        } else {
#pragma unroll
            for (int l = 0; l < kLevels; ++l) {
                const float2 g = interp(fetch_level<false>(l, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight));
                feats[2 * l] = g.x;
                feats[2 * l + 1] = g.y;
            }
        }
    }
    float4* dst = reinterpret_cast<float4*>(a.fscratch + sl * kIn);
#pragma unroll
    for (int q = 0; q < kIn / 4; ++q) dst[q] = make_float4(feats[4 * q], feats[4 * q + 1], feats[4 * q + 2], feats[4 * q + 3]);
}

__global__ void __launch_bounds__(kTcThreads, kCtasPerSm) tex_mlp_kernel(const TextureArgs a, int ppt,
                                                                        int64_t n_tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kOffBar);
    for (int e = tid; e < kHid * kIn / 8; e += kTcThreads) {  // W1 [64][32]
        const int n = e / (kIn / 8), c = e % (kIn / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w1 + n * kIn + c * 8 + i);
        store_split8(smem, kOffW1h, kOffW1l, kmajor_off(n, c * 8, kIn), x);
    }
    for (int e = tid; e < kHid * kHid / 8; e += kTcThreads) {  // W2 [64][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w2 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW2h, kOffW2l, kmajor_off(n, c * 8, kHid), x);
    }
    for (int e = tid; e < kOut * kHid / 8; e += kTcThreads) {  // W3 [48][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w3 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW3h, kOffW3l, kmajor_off(n, c * 8, kHid), x);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kOffTmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kOffTmem);
    uint32_t phase = 0;
    const int K = a.fb.K;
    const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H;
    const int row = tid;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * warp) << 16);
    float* srgb = reinterpret_cast<float*>(smem + kOffRgb);
    constexpr uint32_t kIdesc64 = idesc_bf16_f32(kRows, 64);
    constexpr uint32_t kIdesc48 = idesc_bf16_f32(kRows, 48);
    int n_queries = 0;
    const int p_in = row / K, j_in = row - p_in * K;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t pix = tile * ppt + p_in;
        const bool in_tile = p_in < ppt && pix < npix;
        const int64_t slot = in_tile ? pix * K + j_in : 0;
        const bool valid = in_tile && a.fb.ids[slot] >= 0;
        n_queries += valid;
        float feats[kIn];
        if (valid) {
            const float4* src = reinterpret_cast<const float4*>(a.fscratch + slot * kIn);
#pragma unroll
            for (int q = 0; q < kIn / 4; ++q) {
                const float4 v = src[q];
                feats[4 * q] = v.x;
                feats[4 * q + 1] = v.y;
                feats[4 * q + 2] = v.z;
                feats[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kIn; ++i) feats[i] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < kIn / 8; ++c) store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 8 * c, kIn), feats + 8 * c);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) issue_layer(smem, tmem, kOffW1h, kOffW1l, kIn, kIdesc64, bar);
        // the pixel ray of this row while layer 1 runs
        double dir[3] = {0.0, 0.0, 1.0};
        if (in_tile) pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int layer = 0; layer < 2; ++layer) {
#if NX_TMEM_BATCH
            {
                uint32_t r[kHid];
                tmem_ld_batch<kHid / 16>(taddr, r);
#pragma unroll
                for (int c = 0; c < kHid / 8; ++c) {
                    float v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = fmaxf(__uint_as_float(r[8 * c + i]), 0.f);
                    store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 8 * c, kHid), v);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < kHid / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c, kHid), v);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c + 8, kHid), v + 8);
            }
#endif
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                if (layer == 0) issue_layer(smem, tmem, kOffW2h, kOffW2l, kHid, kIdesc64, bar);
                else issue_layer(smem, tmem, kOffW3h, kOffW3l, kHid, kIdesc48, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        {
            const float x = static_cast<float>(dir[0]), y = static_cast<float>(dir[1]), z = static_cast<float>(dir[2]);
            float b[16];
            sh_basis_f32(x, y, z, b);
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
            for (int c = 0; c < kOut / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int o = 16 * c + i, k = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v[i], b[k], c0);
                    else if (o % 3 == 1) c1 = fmaf(v[i], b[k], c1);
                    else c2 = fmaf(v[i], b[k], c2);
                }
            }
            float rgb[3] = {0.f, 0.f, 0.f};
            if (valid) {
                rgb[0] = fmaxf(0.5f + c0, 0.f);
                rgb[1] = fmaxf(0.5f + c1, 0.f);
                rgb[2] = fmaxf(0.5f + c2, 0.f);
            }
            srgb[row * 3 + 0] = rgb[0];
            srgb[row * 3 + 1] = rgb[1];
            srgb[row * 3 + 2] = rgb[2];
            if (in_tile) {
                a.fb.texture[slot * 3 + 0] = rgb[0];
                a.fb.texture[slot * 3 + 1] = rgb[1];
                a.fb.texture[slot * 3 + 2] = rgb[2];
            }
        }
        tc_fence_before();
        __syncthreads();
        // Eq. 7: final = base + sum_j W[p,j] * texture[p,j] (renderer.cpp:219-236)
        if (tid < ppt) {
            const int64_t qp = tile * ppt + tid;
            if (qp < npix) {
                double acc0 = a.fb.base[qp * 3 + 0], acc1 = a.fb.base[qp * 3 + 1], acc2 = a.fb.base[qp * 3 + 2];
                for (int j = 0; j < K; ++j) {
                    const int64_t sl = qp * K + j;
                    if (a.fb.ids[sl] < 0) continue;
                    const double w = a.fb.weights[sl];
                    const float* tc = srgb + (tid * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
                a.fb.final_img[qp * 3 + 0] = static_cast<float>(acc0);
                a.fb.final_img[qp * 3 + 1] = static_cast<float>(acc1);
                a.fb.final_img[qp * 3 + 2] = static_cast<float>(acc2);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_queries += __shfl_down_sync(0xffffffffu, n_queries, o);
    if ((tid & 31) == 0 && n_queries) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_queries));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------- warp-specialised variant
// One persistent CTA per SM; the pass of a tile (128 rows = 128/K pixels x K slots of a
// bw x bh pixel block) flows through three roles that run concurrently on different
// tiles, handing buffers over with mbarriers:
//   gather warps (16; two groups of 8, alternate tiles): per row, 8 of the 16 levels per
//     thread (two threads per row), features -> bf16 hi/lo split -> the tile's smem A
//     buffer (K-major), fence.proxy.async, arrive `full`;
//   MMA warp (1 elected thread): layer 1 (A1 . W1^T), layer 2, layer 3 into the tile's
//     64-column TMEM slot, one tcgen05.commit per layer to the slot's `done` barrier;
//   epilogue warps (4, one TMEM lane each): D1 -> relu -> split -> A2 in the same smem
//     buffer, arrive `a_ready`; D2 -> A3 likewise; D3 -> SH colour -> texture, Eq. 7,
//     then free the TMEM slot and the buffer for the next tiles.
// Step k of the MMA warp issues L3(k-2), L2(k-1), L1(k); step k of the epilogue drains
// them in the same order, so three tiles are in the tensor-core pipeline while two more
// are gathered. Five 32 KB A buffers + the weights: ~197 KB of shared memory; three TMEM
// slots (192 of 256 allocated columns). No feature scratch goes through HBM.
// Layout per producer mode: kGather = the gather warps above; kBulk = one producer warp
// that copies tiles of pre-gathered, pre-split features (tex_features_img_kernel) with
// the bulk-copy engine (cp.async.bulk, mbarrier transaction counts).
enum WsMode { kGather = 0, kBulk = 1 };
template <int kMode>
struct WsCfg {
    static constexpr int NB = kMode == kGather ? 5 : 4;  // smem A buffers (tiles between producer and epilogue)
    static constexpr int kProducerWarps = kMode == kGather ? 16 : 1;
#ifndef NX_WS_EPI_GROUPS
#define NX_WS_EPI_GROUPS 4
#endif
    static constexpr int kEpiGroups = kMode == kGather ? 1 : NX_WS_EPI_GROUPS;  // 4-warp epilogue groups
    static constexpr int kSlots = kMode == kGather ? 3 : 2 * NX_WS_EPI_GROUPS;   // TMEM slots of 64 columns
    static constexpr int kTmemCols = kSlots * 64 <= 256 ? 256 : 512;
    static constexpr int kMmaWarp = 4 * kEpiGroups;
    static constexpr int kThreads = (kMmaWarp + 1 + kProducerWarps) * 32;  // 672 / 352
    static constexpr int kOffRgb = kOffAh + NB * 2 * kRows * kHid * 2;  // after the weights + A buffers
    static constexpr int kOffBar = kOffRgb + kEpiGroups * 2 * kRows * 3 * 4;
    static constexpr int kNumBars = 3 * NB + 2 * kSlots;  // full, empty, a_ready [NB]; done, tmem_free [slots]
    static constexpr int kOffTmem = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffTmem + 16;
    static_assert(kSmem <= 227 * 1024, "one CTA per SM");
};
constexpr int kWsBufBytes = 2 * kRows * kHid * 2;  // hi + lo, 64-wide bf16: 32 KB
constexpr int kWsOffBuf = kOffAh;                  // = 36 KB (after the weights)
constexpr int kImgBytes = 2 * kRows * kIn * 2;     // a tile's pre-split features: hi 8 KB + lo 8 KB
static_assert(kOffW3l + kOut * kHid * 2 == kWsOffBuf, "weights precede the A buffers");

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void named_barrier_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Issues one layer from buffer offset `abuf` (hi at +0, lo at +16 KB).
__device__ __forceinline__ void ws_issue_layer(uint8_t* smem, uint32_t dtm, int abuf, int off_bh, int off_bl, int K,
                                               uint32_t idesc, uint32_t bar) {
    const uint32_t ah = smem_u32(smem + abuf), al = smem_u32(smem + abuf + kRows * kHid * 2);
    const uint32_t bh = smem_u32(smem + off_bh), bl = smem_u32(smem + off_bl);
    const uint32_t sbo = 16 * K;
    for (int s = 0; s < K / 16; ++s) {
        const uint32_t o = s * 256;
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, s > 0);
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bl + o, 128, sbo), idesc, 1);
        mma_bf16(dtm, smem_desc(al + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, 1);
    }
    mma_commit(bar);
}

struct WsTile {  // row -> slot of local tile k
    int px, py, p_in;
    bool in_tile;
    int64_t slot;
};

__device__ __forceinline__ WsTile ws_tile(int64_t tile, int row, int K, int bw, int bh, int tiles_x, int W, int H) {
    WsTile t;
    const int tpx = static_cast<int>(tile % tiles_x) * bw, tpy = static_cast<int>(tile / tiles_x) * bh;
    t.p_in = row / K;
    const int j = row - t.p_in * K;
    t.px = tpx + t.p_in % bw;
    t.py = tpy + t.p_in / bw;
    t.in_tile = t.p_in < bw * bh && t.px < W && t.py < H;
    t.slot = t.in_tile ? (static_cast<int64_t>(t.py) * W + t.px) * K + j : 0;
    return t;
}

template <int kMode>
__global__ void __launch_bounds__(WsCfg<kMode>::kThreads, 1)
    texture_ws_kernel(const TextureArgs a, const TcConst cst, int bw, int bh, int tiles_x, int64_t n_tiles) {
    using Cfg = WsCfg<kMode>;
    constexpr int kWsNB = Cfg::NB;
    constexpr int kWsThreads = Cfg::kThreads;
    constexpr int kWsOffRgb = Cfg::kOffRgb;
    constexpr int kWsOffTmem = Cfg::kOffTmem;
    constexpr int kWsSlots = Cfg::kSlots;
    constexpr int kG = Cfg::kEpiGroups;
    constexpr int kMmaWarp = Cfg::kMmaWarp;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bars = smem_u32(smem + Cfg::kOffBar);
    auto full = [&](int b) { return bars + 8u * b; };
    auto empty = [&](int b) { return bars + 8u * (kWsNB + b); };
    auto a_ready = [&](int b) { return bars + 8u * (2 * kWsNB + b); };
    auto done = [&](int sl) { return bars + 8u * (3 * kWsNB + sl); };
    auto tmem_free = [&](int sl) { return bars + 8u * (3 * kWsNB + kWsSlots + sl); };

    // ---- setup: weights -> smem (bf16 hi/lo), barriers, TMEM
    for (int e = tid; e < kHid * kIn / 8; e += kWsThreads) {
        const int n = e / (kIn / 8), c = e % (kIn / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w1 + n * kIn + c * 8 + i);
        store_split8(smem, kOffW1h, kOffW1l, kmajor_off(n, c * 8, kIn), x);
    }
    for (int e = tid; e < kHid * kHid / 8; e += kWsThreads) {
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w2 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW2h, kOffW2l, kmajor_off(n, c * 8, kHid), x);
    }
    for (int e = tid; e < kOut * kHid / 8; e += kWsThreads) {
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w3 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW3h, kOffW3l, kmajor_off(n, c * 8, kHid), x);
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kWsOffTmem)),
                     "r"(Cfg::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int b = 0; b < kWsNB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(full(b)),
                         "r"(kMode == kGather ? 32 * Cfg::kProducerWarps / 2 : 1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty(b)), "r"(kRows));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a_ready(b)), "r"(kRows));
        }
        for (int sl = 0; sl < kWsSlots; ++sl) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(done(sl)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tmem_free(sl)), "r"(kRows));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kWsOffTmem);

    const int K = a.fb.K, W = a.cam.W, H = a.cam.H;
    const int64_t n_local = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto tile_of = [&](int64_t k) { return static_cast<int64_t>(blockIdx.x) + k * gridDim.x; };
    auto buf_off = [&](int64_t k) { return kWsOffBuf + static_cast<int>(k % kWsNB) * kWsBufBytes; };
    constexpr int kLoOff = kRows * kHid * 2;  // lo half of a buffer

    if (kMode == kBulk && warp == kMmaWarp + 1) {
        // ================= producer warp: bulk copies of the pre-split feature tiles
        if (lane == 0) {
            const uint8_t* img = reinterpret_cast<const uint8_t*>(a.fscratch);
            for (int64_t k = 0; k < n_local; ++k) {
                const int b = static_cast<int>(k % kWsNB);
                mbar_wait(empty(b), static_cast<uint32_t>(((k / kWsNB) & 1) ^ 1));
                const uint8_t* src = img + tile_of(k) * kImgBytes;
                const uint32_t dst = smem_u32(smem + buf_off(k));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(b)), "r"(kImgBytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "l"(src), "r"(kImgBytes / 2), "r"(full(b))
                    : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dst + kLoOff),
                    "l"(src + kImgBytes / 2), "r"(kImgBytes / 2), "r"(full(b))
                    : "memory");
            }
        }
        __syncwarp();
    } else if (kMode == kGather && warp > kMmaWarp) {
        // ================= gather warps
        const int gw = warp - kMmaWarp - 1, group = gw >> 3, t = (gw & 7) * 32 + lane;
        const int row = t & (kRows - 1), half = t >> 7;
        const uint32_t T = 1u << a.scene.field.log2_table, mask = T - 1u;
        const float2* tab = reinterpret_cast<const float2*>(a.scene.table);
        for (int64_t k = group; k < n_local; k += 2) {
            const int b = static_cast<int>(k % kWsNB);
            mbar_wait(empty(b), static_cast<uint32_t>(((k / kWsNB) & 1) ^ 1));
            const WsTile wt = ws_tile(tile_of(k), row, K, bw, bh, tiles_x, W, H);
            float feats[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) feats[i] = 0.f;
            if (wt.in_tile && a.fb.ids[wt.slot] >= 0) {
                double dir[3];
                pixel_dir(a.cam, wt.px + 0.5, wt.py + 0.5, dir);
                const double tq = a.fb.depths[wt.slot];
                const double x0 = a.cam.o[0] + tq * dir[0];  // build_queries (renderer.cpp:196-198)
                const double x1 = a.cam.o[1] + tq * dir[1];
                const double x2 = a.cam.o[2] + tq * dir[2];
                const float ft = static_cast<float>(a.cam.fx / tq);
                const int l0 = half * 8;
                const bool small =
                    fmax(fabs(x0), fmax(fabs(x1), fabs(x2))) * cst.level_scale[kLevels - 1] < 1073741824.0;
                if (small) {
                    LevelFetch cur = fetch_level<true>(l0, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
#pragma unroll
                    for (int l = 0; l < 8; ++l) {
                        LevelFetch nxt;
                        if (l + 1 < 8)
                            nxt = fetch_level<true>(l0 + l + 1, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
                        const float2 g = interp(cur);
                        feats[2 * l] = g.x;
                        feats[2 * l + 1] = g.y;
                        if (l + 1 < 8) cur = nxt;
                    }
                } else {
#pragma unroll
                    for (int l = 0; l < 8; ++l) {
                        const float2 g = interp(
                            fetch_level<false>(l0 + l, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight));
                        feats[2 * l] = g.x;
                        feats[2 * l + 1] = g.y;
                    }
                }
            }
            const int ab = buf_off(k);
            store_split8(smem, ab, ab + kLoOff, kmajor_off(row, 16 * half, kIn), feats);
            store_split8(smem, ab, ab + kLoOff, kmajor_off(row, 16 * half + 8, kIn), feats + 8);
            fence_async_smem();
            mbar_arrive(full(b));
        }
    } else if (warp == kMmaWarp) {
        // ================= MMA warp (one elected thread issues)
        if (lane == 0) {
            constexpr uint32_t kIdesc64 = idesc_bf16_f32(kRows, 64);
            constexpr uint32_t kIdesc48 = idesc_bf16_f32(kRows, 48);
            for (int64_t k = 0; k < n_local + 2; ++k) {
                const int64_t k3 = k - 2, k2 = k - 1;
                if (k3 >= 0 && k3 < n_local) {  // L3(k-2): A3 written by conv2
                    mbar_wait(a_ready(static_cast<int>(k3 % kWsNB)), 1);
                    tc_fence_after();
                    ws_issue_layer(smem, tmem + 64u * static_cast<uint32_t>(k3 % kWsSlots), buf_off(k3), kOffW3h,
                                   kOffW3l, kHid, kIdesc48, done(static_cast<int>(k3 % kWsSlots)));
                }
                if (k2 >= 0 && k2 < n_local) {  // L2(k-1): A2 written by conv1
                    mbar_wait(a_ready(static_cast<int>(k2 % kWsNB)), 0);
                    tc_fence_after();
                    ws_issue_layer(smem, tmem + 64u * static_cast<uint32_t>(k2 % kWsSlots), buf_off(k2), kOffW2h,
                                   kOffW2l, kHid, kIdesc64, done(static_cast<int>(k2 % kWsSlots)));
                }
                if (k < n_local) {  // L1(k): features gathered, TMEM slot released by final(k-3)
                    mbar_wait(tmem_free(static_cast<int>(k % kWsSlots)), static_cast<uint32_t>(((k / kWsSlots) & 1) ^ 1));
                    mbar_wait(full(static_cast<int>(k % kWsNB)), static_cast<uint32_t>((k / kWsNB) & 1));
                    tc_fence_after();
                    ws_issue_layer(smem, tmem + 64u * static_cast<uint32_t>(k % kWsSlots), buf_off(k), kOffW1h,
                                   kOffW1l, kIn, kIdesc64, done(static_cast<int>(k % kWsSlots)));
                }
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue warps (group g = warp / 4 takes the tiles k = g mod kG;
        // TMEM lanes 32 (warp % 4) .. + 31; row = tid % 128)
        const int g = warp >> 2;
        const int row = tid & (kRows - 1);
        const uint32_t lane_addr = static_cast<uint32_t>(32 * (warp & 3)) << 16;
        float* srgb_base = reinterpret_cast<float*>(smem + kWsOffRgb) + g * 2 * kRows * 3;
        const int ppt = bw * bh;
        int n_queries = 0;
        // completion parity of the i-th layer (0, 1, 2) of local tile k on its TMEM slot
        auto done_parity = [&](int64_t k, int i) { return static_cast<uint32_t>((3 * (k / kWsSlots) + i) & 1); };
        auto conv = [&](int64_t k, int layer) {  // D(layer) -> relu -> split -> A(layer + 1) in k's buffer
            const int sl = static_cast<int>(k % kWsSlots);
            mbar_wait(done(sl), done_parity(k, layer));
            tc_fence_after();
            const uint32_t taddr = tmem + 64u * static_cast<uint32_t>(sl) + lane_addr;
            const int ab = buf_off(k);
#pragma unroll
            for (int c = 0; c < kHid / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
                store_split8(smem, ab, ab + kLoOff, kmajor_off(row, 16 * c, kHid), v);
                store_split8(smem, ab, ab + kLoOff, kmajor_off(row, 16 * c + 8, kHid), v + 8);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(a_ready(static_cast<int>(k % kWsNB)));
        };
        for (int64_t k = 0; k < n_local + 2; ++k) {
            const int64_t k3 = k - 2, k2 = k - 1;
            if (k3 >= 0 && k3 < n_local && k3 % kG == g) {  // final(k-2): D3 -> SH colour -> texture, Eq. 7
                const int sl = static_cast<int>(k3 % kWsSlots);
                mbar_wait(done(sl), done_parity(k3, 2));
                tc_fence_after();
                mbar_arrive(empty(static_cast<int>(k3 % kWsNB)));  // A3 consumed: the buffer is free
                const int64_t tile = tile_of(k3);
                const WsTile wt = ws_tile(tile, row, K, bw, bh, tiles_x, W, H);
                const bool valid = wt.in_tile && a.fb.ids[wt.slot] >= 0;
                n_queries += valid;
                double dir[3] = {0.0, 0.0, 1.0};
                if (wt.in_tile) pixel_dir(a.cam, wt.px + 0.5, wt.py + 0.5, dir);
                float b[16];
                sh_basis_f32(static_cast<float>(dir[0]), static_cast<float>(dir[1]), static_cast<float>(dir[2]), b);
                const uint32_t taddr = tmem + 64u * static_cast<uint32_t>(sl) + lane_addr;
                float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
                for (int c = 0; c < kOut / 16; ++c) {
                    float v[16];
                    tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int o = 16 * c + i, kk = o / 3;
                        if (o % 3 == 0) c0 = fmaf(v[i], b[kk], c0);
                        else if (o % 3 == 1) c1 = fmaf(v[i], b[kk], c1);
                        else c2 = fmaf(v[i], b[kk], c2);
                    }
                }
                tc_fence_before();
                mbar_arrive(tmem_free(sl));  // D3 read: the slot is free for L1(k + 1)
                float rgb[3] = {0.f, 0.f, 0.f};
                if (valid) {
                    rgb[0] = fmaxf(0.5f + c0, 0.f);
                    rgb[1] = fmaxf(0.5f + c1, 0.f);
                    rgb[2] = fmaxf(0.5f + c2, 0.f);
                }
                float* srgb = srgb_base + ((k3 / kG) & 1) * kRows * 3;
                srgb[row * 3 + 0] = rgb[0];
                srgb[row * 3 + 1] = rgb[1];
                srgb[row * 3 + 2] = rgb[2];
                if (wt.in_tile) {
                    a.fb.texture[wt.slot * 3 + 0] = rgb[0];
                    a.fb.texture[wt.slot * 3 + 1] = rgb[1];
                    a.fb.texture[wt.slot * 3 + 2] = rgb[2];
                }
                named_barrier_sync(1 + g, kRows);
                // Eq. 7: final = base + sum_j W[p,j] * texture[p,j] (renderer.cpp:219-236)
                if (row < ppt) {
                    const int tpx = static_cast<int>(tile % tiles_x) * bw, tpy = static_cast<int>(tile / tiles_x) * bh;
                    const int qx = tpx + row % bw, qy = tpy + row / bw;
                    if (qx < W && qy < H) {
                        const int64_t pix = static_cast<int64_t>(qy) * W + qx;
                        double acc0 = a.fb.base[pix * 3 + 0], acc1 = a.fb.base[pix * 3 + 1],
                               acc2 = a.fb.base[pix * 3 + 2];
                        for (int j = 0; j < K; ++j) {
                            const int64_t q = pix * K + j;
                            if (a.fb.ids[q] < 0) continue;
                            const double w = a.fb.weights[q];
                            const float* tc = srgb + (row * K + j) * 3;
                            acc0 += w * tc[0];
                            acc1 += w * tc[1];
                            acc2 += w * tc[2];
                        }
                        a.fb.final_img[pix * 3 + 0] = static_cast<float>(acc0);
                        a.fb.final_img[pix * 3 + 1] = static_cast<float>(acc1);
                        a.fb.final_img[pix * 3 + 2] = static_cast<float>(acc2);
                    }
                }
            }
            if (k2 >= 0 && k2 < n_local && k2 % kG == g) conv(k2, 1);  // D2 -> A3
            if (k < n_local && k % kG == g) conv(k, 0);                // D1 -> A2
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_queries += __shfl_down_sync(0xffffffffu, n_queries, o);
        if (lane == 0 && n_queries) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_queries));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMmaWarp)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
}

// The gathers of the bulk-fed variant: one thread per slot at full occupancy, features
// split into bf16 hi / lo and stored as the tile's K-major operand image (16 KB per
// 128-row tile: hi then lo), at the (tile, row) texture_ws_kernel<kBulk> assigns the slot.
#ifndef NX_FEAT_MINB
#define NX_FEAT_MINB 6  // 80 registers, 6 CTAs per SM (measured: 2.257 -> 2.250 ms per frame; final build: 5 481.8, 6 488.5, 8 470.5 frames/s)
#endif
#ifdef NX_FEAT_MINB
#define NX_FEAT_BOUNDS __launch_bounds__(128, NX_FEAT_MINB)
#else
#define NX_FEAT_BOUNDS __launch_bounds__(128)
#endif
__global__ void NX_FEAT_BOUNDS tex_features_img_kernel(const TextureArgs a, const TcConst cst, int bw, int bh,
                                                               int tiles_x) {
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int K = a.fb.K;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
    if (sl >= total) return;
    float feats[kIn];
#pragma unroll
    for (int i = 0; i < kIn; ++i) feats[i] = 0.f;
    const int64_t pix = sl / K;
    const int j = static_cast<int>(sl - pix * K);
    const int px = static_cast<int>(pix % a.cam.W), py = static_cast<int>(pix / a.cam.W);
    if (a.fb.ids[sl] >= 0) {
        double dir[3];
        pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
        const double t = a.fb.depths[sl];
        const double x0 = a.cam.o[0] + t * dir[0], x1 = a.cam.o[1] + t * dir[1], x2 = a.cam.o[2] + t * dir[2];
        const float ft = static_cast<float>(a.cam.fx / t);
        const uint32_t T = 1u << a.scene.field.log2_table, mask = T - 1u;
        const float2* tab = reinterpret_cast<const float2*>(a.scene.table);
        const bool small = fmax(fabs(x0), fmax(fabs(x1), fabs(x2))) * cst.level_scale[kLevels - 1] < 1073741824.0;
        if (small) {
            LevelFetch cur = fetch_level<true>(0, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
#pragma unroll
            for (int l = 0; l < kLevels; ++l) {
                LevelFetch nxt;
                if (l + 1 < kLevels) nxt = fetch_level<true>(l + 1, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
                const float2 g = interp(cur);
                feats[2 * l] = g.x;
                feats[2 * l + 1] = g.y;
                if (l + 1 < kLevels) cur = nxt;
            }
        } else {
#pragma unroll
            for (int l = 0; l < kLevels; ++l) {
                const float2 g = interp(fetch_level<false>(l, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight));
                feats[2 * l] = g.x;
                feats[2 * l + 1] = g.y;
            }
        }
    }
    const int64_t tile = static_cast<int64_t>(py / bh) * tiles_x + px / bw;
    const int row = ((py % bh) * bw + px % bw) * K + j;
    uint8_t* img = reinterpret_cast<uint8_t*>(a.fscratch) + tile * kImgBytes;
#pragma unroll
    for (int c = 0; c < kIn / 8; ++c) store_split8(img, 0, kImgBytes / 2, kmajor_off(row, 8 * c, kIn), feats + 8 * c);
}


// ---------------------------------------------------------------- split2: bulk-fed decoder
// The split pass with the gathers writing pre-split operand tiles (tex_features_img_kernel)
// and a single-role decoder that streams them with the bulk-copy engine: while a tile's
// three layers run, the next tile's 16 KB operand image lands in the other of two
// buffers (cp.async.bulk + mbarrier transaction count); layer 1 reads it in place (no
// register round trip, no split on this side). Two 128-thread CTAs per SM (~101 KB).
#ifndef NX_TMEM_BATCH
#define NX_TMEM_BATCH 1
#endif
constexpr int kB2OffImg = kOffAh + 2 * kRows * kHid * 2;        // after the 64-wide A operand
constexpr int kB2OffRgb = kB2OffImg + 2 * kImgBytes;             // two image buffers
constexpr int kB2OffBar = kB2OffRgb + kRows * 3 * 4;             // mma, full[2]
constexpr int kB2OffTmem = kB2OffBar + 3 * 8;
constexpr int kB2Smem = kB2OffTmem + 8;
static_assert(kB2Smem <= 113 * 1024, "two CTAs per SM");

__device__ __forceinline__ void b2_issue_layer(uint8_t* smem, uint32_t dtm, int a_hi, int a_lo, int off_bh, int off_bl,
                                               int K, uint32_t idesc, uint32_t bar) {
    const uint32_t ah = smem_u32(smem + a_hi), al = smem_u32(smem + a_lo);
    const uint32_t bh = smem_u32(smem + off_bh), bl = smem_u32(smem + off_bl);
    const uint32_t sbo = 16 * K;
    for (int s = 0; s < K / 16; ++s) {
        const uint32_t o = s * 256;
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, s > 0);
        mma_bf16(dtm, smem_desc(ah + o, 128, sbo), smem_desc(bl + o, 128, sbo), idesc, 1);
        mma_bf16(dtm, smem_desc(al + o, 128, sbo), smem_desc(bh + o, 128, sbo), idesc, 1);
    }
    mma_commit(bar);
}

#ifndef NX_B2_MINB
#define NX_B2_MINB 2
#endif
__global__ void __launch_bounds__(kTcThreads, NX_B2_MINB) tex_mlp_bulk_kernel(const TextureArgs a, int bw, int bh, int tiles_x,
                                                                   int64_t n_tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kB2OffBar);
    auto full = [&](int b) { return smem_u32(smem + kB2OffBar + 8 * (1 + b)); };
    for (int e = tid; e < kHid * kIn / 8; e += kTcThreads) {  // W1 [64][32]
        const int n = e / (kIn / 8), c = e % (kIn / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w1 + n * kIn + c * 8 + i);
        store_split8(smem, kOffW1h, kOffW1l, kmajor_off(n, c * 8, kIn), x);
    }
    for (int e = tid; e < kHid * kHid / 8; e += kTcThreads) {  // W2 [64][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w2 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW2h, kOffW2l, kmajor_off(n, c * 8, kHid), x);
    }
    for (int e = tid; e < kOut * kHid / 8; e += kTcThreads) {  // W3 [48][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w3 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW3h, kOffW3l, kmajor_off(n, c * 8, kHid), x);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kB2OffTmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full(0)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full(1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kB2OffTmem);
    uint32_t phase = 0;
    const int K = a.fb.K, W = a.cam.W, H = a.cam.H;
    const int row = tid, ppt = bw * bh;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * warp) << 16);
    float* srgb = reinterpret_cast<float*>(smem + kB2OffRgb);
    constexpr uint32_t kIdesc64 = idesc_bf16_f32(kRows, 64);
    constexpr uint32_t kIdesc48 = idesc_bf16_f32(kRows, 48);
    const uint8_t* img = reinterpret_cast<const uint8_t*>(a.fscratch);
    auto load_tile = [&](int64_t tile, int b) {  // thread 0: the tile's 16 KB image into buffer b
        const uint32_t dst = smem_u32(smem + kB2OffImg + b * kImgBytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(b)), "r"(kImgBytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(img + tile * kImgBytes), "r"(kImgBytes), "r"(full(b))
                     : "memory");
    };
    int n_queries = 0;
    int64_t k = 0;
    if (tid == 0 && blockIdx.x < n_tiles) load_tile(blockIdx.x, 0);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int b = static_cast<int>(k & 1);
        // the other buffer's last reader (the previous tile's layer 1) has completed
        if (tid == 0 && tile + gridDim.x < n_tiles) load_tile(tile + gridDim.x, b ^ 1);
        const WsTile wt = ws_tile(tile, row, K, bw, bh, tiles_x, W, H);
        const bool valid = wt.in_tile && a.fb.ids[wt.slot] >= 0;
        n_queries += valid;
        // Eq. 7 inputs of pixel `row` of the tile, loaded now: their latency hides behind
        // the three layers instead of stalling the tile's end
        constexpr int kPre = 4;
        int64_t e_pix = -1;
        double e_acc[3] = {0.0, 0.0, 0.0}, e_w[kPre];
        int32_t e_id[kPre];
        if (row < ppt) {
            const int qx = static_cast<int>(tile % tiles_x) * bw + row % bw;
            const int qy = static_cast<int>(tile / tiles_x) * bh + row / bw;
            if (qx < W && qy < H) {
                e_pix = static_cast<int64_t>(qy) * W + qx;
                e_acc[0] = a.fb.base[e_pix * 3 + 0];
                e_acc[1] = a.fb.base[e_pix * 3 + 1];
                e_acc[2] = a.fb.base[e_pix * 3 + 2];
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    e_id[j] = j < K ? a.fb.ids[e_pix * K + j] : -1;
                    e_w[j] = j < K ? a.fb.weights[e_pix * K + j] : 0.0;
                }
            }
        }
        mbar_wait(full(b), static_cast<uint32_t>((k >> 1) & 1));
        tc_fence_after();
        const int ib = kB2OffImg + b * kImgBytes;
        if (tid == 0) b2_issue_layer(smem, tmem, ib, ib + kImgBytes / 2, kOffW1h, kOffW1l, kIn, kIdesc64, bar);
        double dir[3] = {0.0, 0.0, 1.0};
        if (wt.in_tile) pixel_dir(a.cam, wt.px + 0.5, wt.py + 0.5, dir);
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int layer = 0; layer < 2; ++layer) {
#if NX_TMEM_BATCH
            {
                uint32_t r[kHid];
                tmem_ld_batch<kHid / 16>(taddr, r);
#pragma unroll
                for (int c = 0; c < kHid / 8; ++c) {
                    float v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = fmaxf(__uint_as_float(r[8 * c + i]), 0.f);
                    store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 8 * c, kHid), v);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < kHid / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c, kHid), v);
                store_split8(smem, kOffAh, kOffAl, kmajor_off(row, 16 * c + 8, kHid), v + 8);
            }
#endif
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                if (layer == 0) b2_issue_layer(smem, tmem, kOffAh, kOffAl, kOffW2h, kOffW2l, kHid, kIdesc64, bar);
                else b2_issue_layer(smem, tmem, kOffAh, kOffAl, kOffW3h, kOffW3l, kHid, kIdesc48, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        {
            float bb[16];
            sh_basis_f32(static_cast<float>(dir[0]), static_cast<float>(dir[1]), static_cast<float>(dir[2]), bb);
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#if NX_TMEM_BATCH
            {
                uint32_t r[kOut];
                tmem_ld_batch<kOut / 16>(taddr, r);
#pragma unroll
                for (int o = 0; o < kOut; ++o) {
                    const float v = __uint_as_float(r[o]);
                    const int kk = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v, bb[kk], c0);
                    else if (o % 3 == 1) c1 = fmaf(v, bb[kk], c1);
                    else c2 = fmaf(v, bb[kk], c2);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < kOut / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int o = 16 * c + i, kk = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v[i], bb[kk], c0);
                    else if (o % 3 == 1) c1 = fmaf(v[i], bb[kk], c1);
                    else c2 = fmaf(v[i], bb[kk], c2);
                }
            }
#endif
            float rgb[3] = {0.f, 0.f, 0.f};
            if (valid) {
                rgb[0] = fmaxf(0.5f + c0, 0.f);
                rgb[1] = fmaxf(0.5f + c1, 0.f);
                rgb[2] = fmaxf(0.5f + c2, 0.f);
            }
            srgb[row * 3 + 0] = rgb[0];
            srgb[row * 3 + 1] = rgb[1];
            srgb[row * 3 + 2] = rgb[2];
            if (wt.in_tile) {
                a.fb.texture[wt.slot * 3 + 0] = rgb[0];
                a.fb.texture[wt.slot * 3 + 1] = rgb[1];
                a.fb.texture[wt.slot * 3 + 2] = rgb[2];
            }
        }
        tc_fence_before();
        __syncthreads();
        // Eq. 7: final = base + sum_j W[p,j] * texture[p,j] (renderer.cpp:219-236)
        if (e_pix >= 0) {
            const int64_t pix = e_pix;
            double acc0 = e_acc[0], acc1 = e_acc[1], acc2 = e_acc[2];
            if (K <= kPre) {
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    if (j >= K || e_id[j] < 0) continue;
                    const double w = e_w[j];
                    const float* tc = srgb + (row * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
            } else {
                for (int j = 0; j < K; ++j) {
                    const int64_t q = pix * K + j;
                    if (a.fb.ids[q] < 0) continue;
                    const double w = a.fb.weights[q];
                    const float* tc = srgb + (row * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
            }
            a.fb.final_img[pix * 3 + 0] = static_cast<float>(acc0);
            a.fb.final_img[pix * 3 + 1] = static_cast<float>(acc1);
            a.fb.final_img[pix * 3 + 2] = static_cast<float>(acc2);
        }
        // srgb and the A operand are rewritten next tile only after its layer-1 wait and
        // the barrier before layer 2, which every thread reaches after this point
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_queries += __shfl_down_sync(0xffffffffu, n_queries, o);
    if ((tid & 31) == 0 && n_queries) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_queries));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// split2ts: the bulk-fed decoder with the hidden activations in tensor memory. The
// epilogue writes the relu'd, bf16-split activations back to TMEM (tcgen05.st) and
// layers 2 / 3 read their A operand from there: no shared-memory A buffer (~70 KB per
// CTA, three CTAs per SM), no generic-to-async proxy fence. TMEM: accumulator columns
// [0, 64), A hi [64, 96), A lo [96, 128).
#ifndef NX_TS_SINGLE
#define NX_TS_SINGLE 1  // one image buffer, refilled once layer 1 has read it (four CTAs per SM)
#endif
constexpr int kTsImgBufs = NX_TS_SINGLE ? 1 : 2;
constexpr int kTsOffImg = kOffAh;                         // the weights, then the image buffer(s)
constexpr int kTsOffRgb = kTsOffImg + kTsImgBufs * kImgBytes;
constexpr int kTsOffBar = kTsOffRgb + kRows * 3 * 4;
constexpr int kTsOffTmem = kTsOffBar + 3 * 8;
constexpr int kTsSmem = kTsOffTmem + 8;
constexpr uint32_t kTsTmemCols = 128;
static_assert(kTsSmem <= (NX_TS_SINGLE ? 56 : 74) * 1024, "four (three) CTAs per SM");

__device__ __forceinline__ void ts_issue_layer(uint32_t dtm, uint32_t a_hi, uint32_t a_lo, uint8_t* smem, int off_bh,
                                               int off_bl, int K, uint32_t idesc, uint32_t bar) {
    const uint32_t bh = smem_u32(smem + off_bh), bl = smem_u32(smem + off_bl);
    const uint32_t sbo = 16 * K;
    for (int s = 0; s < K / 16; ++s) {
        const uint32_t o = s * 256;
        mma_bf16_ts(dtm, a_hi + 8 * s, smem_desc(bh + o, 128, sbo), idesc, s > 0);
        mma_bf16_ts(dtm, a_hi + 8 * s, smem_desc(bl + o, 128, sbo), idesc, 1);
        mma_bf16_ts(dtm, a_lo + 8 * s, smem_desc(bh + o, 128, sbo), idesc, 1);
    }
    mma_commit(bar);
}

#ifndef NX_TS_MINB
#define NX_TS_MINB (NX_TS_SINGLE ? 4 : 3)  // measured: single buffer x 4 CTAs 0.308 ms, two buffers x 3 0.354 (5: 0.46, 453 frames/s)
#endif
__global__ void __launch_bounds__(kTcThreads, NX_TS_MINB) tex_mlp_ts_kernel(const TextureArgs a, int bw, int bh, int tiles_x,
                                                                   int64_t n_tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kTsOffBar);
    auto full = [&](int b) { return smem_u32(smem + kTsOffBar + 8 * (1 + b)); };
    for (int e = tid; e < kHid * kIn / 8; e += kTcThreads) {  // W1 [64][32]
        const int n = e / (kIn / 8), c = e % (kIn / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w1 + n * kIn + c * 8 + i);
        store_split8(smem, kOffW1h, kOffW1l, kmajor_off(n, c * 8, kIn), x);
    }
    for (int e = tid; e < kHid * kHid / 8; e += kTcThreads) {  // W2 [64][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w2 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW2h, kOffW2l, kmajor_off(n, c * 8, kHid), x);
    }
    for (int e = tid; e < kOut * kHid / 8; e += kTcThreads) {  // W3 [48][64]
        const int n = e / (kHid / 8), c = e % (kHid / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(a.scene.w3 + n * kHid + c * 8 + i);
        store_split8(smem, kOffW3h, kOffW3l, kmajor_off(n, c * 8, kHid), x);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kTsOffTmem)),
                     "r"(kTsTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full(0)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full(1)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kTsOffTmem);
    uint32_t phase = 0;
    const int K = a.fb.K, W = a.cam.W, H = a.cam.H;
    const int row = tid, ppt = bw * bh;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(32 * warp) << 16);
    float* srgb = reinterpret_cast<float*>(smem + kTsOffRgb);
    constexpr uint32_t kIdesc64 = idesc_bf16_f32(kRows, 64);
    constexpr uint32_t kIdesc48 = idesc_bf16_f32(kRows, 48);
    const uint8_t* img = reinterpret_cast<const uint8_t*>(a.fscratch);
    auto load_tile = [&](int64_t tile, int b) {  // thread 0: the tile's 16 KB image into buffer b
        const uint32_t dst = smem_u32(smem + kTsOffImg + b * kImgBytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full(b)), "r"(kImgBytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(img + tile * kImgBytes), "r"(kImgBytes), "r"(full(b))
                     : "memory");
    };
    int n_queries = 0;
    int64_t k = 0;
    if (tid == 0 && blockIdx.x < n_tiles) load_tile(blockIdx.x, 0);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int b = NX_TS_SINGLE ? 0 : static_cast<int>(k & 1);
        // the other buffer's last reader (the previous tile's layer 1) has completed
        if (!NX_TS_SINGLE && tid == 0 && tile + gridDim.x < n_tiles) load_tile(tile + gridDim.x, b ^ 1);
        const WsTile wt = ws_tile(tile, row, K, bw, bh, tiles_x, W, H);
        const bool valid = wt.in_tile && a.fb.ids[wt.slot] >= 0;
        n_queries += valid;
        // Eq. 7 inputs of pixel `row` of the tile, loaded now: their latency hides behind
        // the three layers instead of stalling the tile's end
        constexpr int kPre = 4;
        int64_t e_pix = -1;
        double e_acc[3] = {0.0, 0.0, 0.0}, e_w[kPre];
        int32_t e_id[kPre];
        if (row < ppt) {
            const int qx = static_cast<int>(tile % tiles_x) * bw + row % bw;
            const int qy = static_cast<int>(tile / tiles_x) * bh + row / bw;
            if (qx < W && qy < H) {
                e_pix = static_cast<int64_t>(qy) * W + qx;
                e_acc[0] = a.fb.base[e_pix * 3 + 0];
                e_acc[1] = a.fb.base[e_pix * 3 + 1];
                e_acc[2] = a.fb.base[e_pix * 3 + 2];
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    e_id[j] = j < K ? a.fb.ids[e_pix * K + j] : -1;
                    e_w[j] = j < K ? a.fb.weights[e_pix * K + j] : 0.0;
                }
            }
        }
        mbar_wait(full(b), static_cast<uint32_t>(NX_TS_SINGLE ? (k & 1) : ((k >> 1) & 1)));
        tc_fence_after();
        const int ib = kTsOffImg + b * kImgBytes;
        if (tid == 0) b2_issue_layer(smem, tmem, ib, ib + kImgBytes / 2, kOffW1h, kOffW1l, kIn, kIdesc64, bar);
        double dir[3] = {0.0, 0.0, 1.0};
        if (wt.in_tile) pixel_dir(a.cam, wt.px + 0.5, wt.py + 0.5, dir);
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll 1
        for (int layer = 0; layer < 2; ++layer) {
            {
                uint32_t r[kHid];
                tmem_ld_batch<kHid / 16>(taddr, r);
                uint32_t hi[kHid / 2], lo[kHid / 2];
#pragma unroll
                for (int i = 0; i < kHid / 2; ++i) {
                    const float x0 = fmaxf(__uint_as_float(r[2 * i]), 0.f), x1 = fmaxf(__uint_as_float(r[2 * i + 1]), 0.f);
                    hi[i] = pack_bf16(x0, x1);
                    const float h0 = __uint_as_float(hi[i] << 16), h1 = __uint_as_float(hi[i] & 0xffff0000u);
                    lo[i] = pack_bf16(x0 - h0, x1 - h1);
                }
                tmem_st32(taddr + 64, hi);
                tmem_st32(taddr + 96, lo);
                tmem_wait_st();
            }
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
            // single buffer: layer 1 (its only reader) has completed and every thread is past
            // this tile's wait on it (the barrier above), so the next tile's image can land
            if (NX_TS_SINGLE && layer == 0 && tid == 0 && tile + gridDim.x < n_tiles) load_tile(tile + gridDim.x, 0);
            if (tid == 0) {
                if (layer == 0) ts_issue_layer(tmem, tmem + 64, tmem + 96, smem, kOffW2h, kOffW2l, kHid, kIdesc64, bar);
                else ts_issue_layer(tmem, tmem + 64, tmem + 96, smem, kOffW3h, kOffW3l, kHid, kIdesc48, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        {
            float bb[16];
            sh_basis_f32(static_cast<float>(dir[0]), static_cast<float>(dir[1]), static_cast<float>(dir[2]), bb);
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#if NX_TMEM_BATCH
            {
                uint32_t r[kOut];
                tmem_ld_batch<kOut / 16>(taddr, r);
#pragma unroll
                for (int o = 0; o < kOut; ++o) {
                    const float v = __uint_as_float(r[o]);
                    const int kk = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v, bb[kk], c0);
                    else if (o % 3 == 1) c1 = fmaf(v, bb[kk], c1);
                    else c2 = fmaf(v, bb[kk], c2);
                }
            }
#else
#pragma unroll
            for (int c = 0; c < kOut / 16; ++c) {
                float v[16];
                tmem_ld16(taddr + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int o = 16 * c + i, kk = o / 3;
                    if (o % 3 == 0) c0 = fmaf(v[i], bb[kk], c0);
                    else if (o % 3 == 1) c1 = fmaf(v[i], bb[kk], c1);
                    else c2 = fmaf(v[i], bb[kk], c2);
                }
            }
#endif
            float rgb[3] = {0.f, 0.f, 0.f};
            if (valid) {
                rgb[0] = fmaxf(0.5f + c0, 0.f);
                rgb[1] = fmaxf(0.5f + c1, 0.f);
                rgb[2] = fmaxf(0.5f + c2, 0.f);
            }
            srgb[row * 3 + 0] = rgb[0];
            srgb[row * 3 + 1] = rgb[1];
            srgb[row * 3 + 2] = rgb[2];
            if (wt.in_tile) {
                a.fb.texture[wt.slot * 3 + 0] = rgb[0];
                a.fb.texture[wt.slot * 3 + 1] = rgb[1];
                a.fb.texture[wt.slot * 3 + 2] = rgb[2];
            }
        }
        tc_fence_before();
        __syncthreads();
        // Eq. 7: final = base + sum_j W[p,j] * texture[p,j] (renderer.cpp:219-236)
        if (e_pix >= 0) {
            const int64_t pix = e_pix;
            double acc0 = e_acc[0], acc1 = e_acc[1], acc2 = e_acc[2];
            if (K <= kPre) {
#pragma unroll
                for (int j = 0; j < kPre; ++j) {
                    if (j >= K || e_id[j] < 0) continue;
                    const double w = e_w[j];
                    const float* tc = srgb + (row * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
            } else {
                for (int j = 0; j < K; ++j) {
                    const int64_t q = pix * K + j;
                    if (a.fb.ids[q] < 0) continue;
                    const double w = a.fb.weights[q];
                    const float* tc = srgb + (row * K + j) * 3;
                    acc0 += w * tc[0];
                    acc1 += w * tc[1];
                    acc2 += w * tc[2];
                }
            }
            a.fb.final_img[pix * 3 + 0] = static_cast<float>(acc0);
            a.fb.final_img[pix * 3 + 1] = static_cast<float>(acc1);
            a.fb.final_img[pix * 3 + 2] = static_cast<float>(acc2);
        }
        // srgb and the A operand are rewritten next tile only after its layer-1 wait and
        // the barrier before layer 2, which every thread reaches after this point
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_queries += __shfl_down_sync(0xffffffffu, n_queries, o);
    if ((tid & 31) == 0 && n_queries) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_queries));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTsTmemCols));
}

}  // namespace

int texture_tc_path() {
    // Measured at config 2 (ms per frame, two streams / one stream): split2ts 2.21 / 2.42
    // (default; with the collection stream at the higher priority), split2 2.25 / 2.56,
    // and with the earlier round-2 composite split 2.53 / 2.78, bulk-fed warp-specialised
    // with 4 epilogue groups 2.81 / 2.82, gather warp-specialised 3.05 / 3.12. The warp-
    // specialised kernels hold one ~170-200 KB CTA per SM, so the next frame's composite
    // cannot share the SM while they run.
    static const int path = [] {
        const char* e = getenv("NX_TEXTURE_PATH");
        if (e && strcmp(e, "fused") == 0) return 1;
        if (e && strcmp(e, "ws") == 0) return 0;
        if (e && strcmp(e, "bulk") == 0) return 3;
        if (e && strcmp(e, "split") == 0) return 2;
        if (e && strcmp(e, "split2") == 0) return 4;
        return 5;
    }();
    return path;
}

size_t texture_tc_scratch_bytes(int W, int H, int K) {
    if (K <= 0) return 0;
    const int path = texture_tc_path();
    if (path == 2) return static_cast<size_t>(W) * H * K * kIn * sizeof(float);
    if (path != 3 && path != 4 && path != 5) return 0;
    const int ppt = kRows / K;
    const int bw = (kRows % K == 0 && ppt % 8 == 0) ? 8 : ppt;
    const int bh = ppt / bw;
    return static_cast<size_t>((W + bw - 1) / bw) * ((H + bh - 1) / bh) * kImgBytes;
}

bool texture_tc_supported(const nx_field_desc& fd) {
    return fd.levels == kLevels && fd.features == 2 && fd.n_hidden == kHid;
}

int launch_texture_tc(const TextureArgs& a, cudaStream_t s) {
    const int K = a.fb.K;
    // NX_TEXTURE_PATH selects the variant: "split" (default: gathers, then the MLP kernel
    // over a feature scratch), "ws" (warp-specialised, no scratch) or "fused" (one CTA
    // role, three per SM).
    const int path = texture_tc_path();
    if ((path == 0 || ((path == 3 || path == 4 || path == 5) && a.fscratch)) && K > 0) {
        const int ppt = kRows / K;
        const int bw = (kRows % K == 0 && ppt % 8 == 0) ? 8 : ppt;
        const int bh = ppt / bw;
        const int tiles_x = (a.cam.W + bw - 1) / bw;
        const int64_t n_tiles = static_cast<int64_t>(tiles_x) * ((a.cam.H + bh - 1) / bh);
        if (n_tiles == 0) return NX_OK;
        TcConst cst;
        double sc = a.scene.field.base_scale;
        for (int l = 0; l < kLevels; ++l, sc *= a.scene.field.growth) {
            cst.level_scale[l] = sc;
            cst.inv_level_scale[l] = static_cast<float>(1.0 / sc);
        }
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        static const int ws_ctas = [] {  // experiments: CTAs of the warp-specialised kernels
            const char* e = getenv("NX_WS_CTAS");
            return e ? atoi(e) : 0;
        }();
        const int64_t grid = std::min<int64_t>(n_tiles, ws_ctas > 0 ? ws_ctas : sms);
        if (path == 0) {
            cudaFuncSetAttribute(texture_ws_kernel<kGather>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 WsCfg<kGather>::kSmem);
            count_launch();
            texture_ws_kernel<kGather><<<static_cast<unsigned>(grid), WsCfg<kGather>::kThreads, WsCfg<kGather>::kSmem,
                                         s>>>(a, cst, bw, bh, tiles_x, n_tiles);
            return NX_OK;
        }
        const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
        count_launch(2);
        tex_features_img_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s>>>(a, cst, bw, bh, tiles_x);
        if (a.ev_mid) {
            cudaEventRecord(a.ev_mid, s);
            a.ev_mid_recorded = true;
        }
        if (path == 5) {  // split2ts: activations in tensor memory, four CTAs per SM
            cudaFuncSetAttribute(tex_mlp_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTsSmem);
            static const int per_sm = [] {  // resident decoder CTAs per SM (shared with the composite)
                const char* e = getenv("NX_TS_CTAS_PER_SM");
                return e ? std::max(1, atoi(e)) : NX_TS_MINB;
            }();
            const int64_t g3 = std::min<int64_t>(n_tiles, per_sm * static_cast<int64_t>(sms));
            tex_mlp_ts_kernel<<<static_cast<unsigned>(g3), kTcThreads, kTsSmem, s>>>(a, bw, bh, tiles_x, n_tiles);
            return NX_OK;
        }
        if (path == 4) {  // split2: the single-role decoder fed by bulk copies, two CTAs per SM
            cudaFuncSetAttribute(tex_mlp_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kB2Smem);
            const int64_t g2 = std::min<int64_t>(n_tiles, 2 * static_cast<int64_t>(sms));
            tex_mlp_bulk_kernel<<<static_cast<unsigned>(g2), kTcThreads, kB2Smem, s>>>(a, bw, bh, tiles_x, n_tiles);
            return NX_OK;
        }
        cudaFuncSetAttribute(texture_ws_kernel<kBulk>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             WsCfg<kBulk>::kSmem);
        texture_ws_kernel<kBulk><<<static_cast<unsigned>(grid), WsCfg<kBulk>::kThreads, WsCfg<kBulk>::kSmem, s>>>(
            a, cst, bw, bh, tiles_x, n_tiles);
        return NX_OK;
    }
    if (a.fscratch && path == 2) {  // split: gathers at full occupancy, then the tensor-core MLP
        const int ppt = kRows / K;
        const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H, total = npix * K;
        if (total == 0) return NX_OK;
        const int64_t n_tiles = (npix + ppt - 1) / ppt;
        TcConst cst;
        double sc = a.scene.field.base_scale;
        for (int l = 0; l < kLevels; ++l, sc *= a.scene.field.growth) {
            cst.level_scale[l] = sc;
            cst.inv_level_scale[l] = static_cast<float>(1.0 / sc);
        }
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(tex_mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemUsed);
        count_launch(2);
        tex_features_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s>>>(a, cst, total);
        if (a.ev_mid) {
            cudaEventRecord(a.ev_mid, s);
            a.ev_mid_recorded = true;
        }
        static const int mlp_per_sm = [] {  // decoder CTAs per SM (NX_MLP_CTAS_PER_SM, experiments)
            const char* e = getenv("NX_MLP_CTAS_PER_SM");
            const int v = e ? atoi(e) : kCtasPerSm;
            return v < 1 ? 1 : (v > kCtasPerSm ? kCtasPerSm : v);
        }();
        const int64_t grid = std::min<int64_t>(n_tiles, static_cast<int64_t>(mlp_per_sm) * sms);
        tex_mlp_kernel<<<static_cast<unsigned>(grid), kTcThreads, kSmemUsed, s>>>(a, ppt, n_tiles);
        return NX_OK;
    }
    // Tiles are pixel blocks (8 wide) so that neighbouring rows query neighbouring
    // lattice cells; K that do not divide 128 use a one-row block of 128/K pixels.
    const int ppt = kRows / K;
    const int bw = (kRows % K == 0 && ppt % 8 == 0) ? 8 : ppt;
    const int bh = ppt / bw;
    const int tiles_x = (a.cam.W + bw - 1) / bw;
    const int64_t n_tiles = static_cast<int64_t>(tiles_x) * ((a.cam.H + bh - 1) / bh);
    if (n_tiles == 0) return NX_OK;
    TcConst cst;
    double sc = a.scene.field.base_scale;
    for (int l = 0; l < kLevels; ++l, sc *= a.scene.field.growth) {
        cst.level_scale[l] = sc;
        cst.inv_level_scale[l] = static_cast<float>(1.0 / sc);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(texture_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemUsed);
    // Persistent CTAs on every slot (measured best: 3/SM 273 FPS vs 2/SM 265 FPS at
    // config 2, profiles/r01); NX_TEXTURE_CTAS_PER_SM overrides for experiments.
    static const int per_sm = [] {
        const char* e = getenv("NX_TEXTURE_CTAS_PER_SM");
        const int v = e ? atoi(e) : kCtasPerSm;
        return v < 1 ? 1 : (v > kCtasPerSm ? kCtasPerSm : v);
    }();
    const int64_t grid = std::min<int64_t>(n_tiles, static_cast<int64_t>(per_sm) * sms);
    count_launch();
    texture_tc_kernel<<<static_cast<unsigned>(grid), kTcThreads, kSmemUsed, s>>>(a, cst, bw, bh, tiles_x, n_tiles);
    return NX_OK;
}

}  // namespace nx
