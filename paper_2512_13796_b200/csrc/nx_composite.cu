// K6 composite: per-tile front-to-back alpha compositing with early termination
// and a top-K buffer (collection_pass, renderer.cpp:115-171).
//
// One 64-thread CTA per 8x8-pixel work tile (two warps of 8x4 pixels), one thread
// per pixel: many small CTAs per SM keep the load balanced across tiles whose hit
// counts differ a lot. The tile's work list (ids in (depth, id) order) is walked in
// chunks whose fp32 prefilter records are staged in shared memory (broadcast reads).
// Per chunk, each warp
//   0. compacts the chunk to the primitives whose padded pixel rect meets its 8x4
//      block (warp ballots, list order kept), then per group of kSub of those:
//   S. starts asynchronous copies (cp.async) of the group's fp64 exact records and SH
//      coefficients into its private shared staging — they land while A runs;
//   A. tests each pixel against the primitive's pixel rect and prefilters in fp32
//      (conservative): a pair is dropped only if it provably fails the
//      reference's t > near_eps or |u| <= ru, |v| <= rv conditions (hence alpha < 1/255);
//   B1. pools the survivors of its 32 pixels and evaluates them with all lanes busy on
//      the exact fp64 path — the reference's intersect() formulas (intersect.hpp:23-42)
//      and eval_kernel (kernel.hpp:16-30, table-driven exp / log: nx_fastmath.cuh) —
//      plus the primitive's SH colour (fp32, colour only), all from the staging;
//   B2. composites, per pixel and in list order, its own survivors: alpha clamp,
//      weight, top-K insert, transmittance update and termination
//      (renderer.cpp:144-153), all fp64.
// Every decision is the reference's, taken in fp64 with its formulas; culling and
// prefilter only skip provable misses, so contributor lists are bit-exact.
#include "nx_composite.cuh"
#include "nx_fastmath.cuh"

#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

namespace nx {

namespace {

constexpr int kThreads = kWorkTile * kWorkTile;  // 64: one thread per pixel of the work tile
constexpr int kWarps = kThreads / 32;
#ifndef NX_COMPOSITE_CHUNK
// 48: the certified CTA drops to ~17.4 KB of shared memory and 12 CTAs fit per SM (work
// lists average ~63 primitives per 8x8 tile). Measured (frames/s, 200 frames): 32 at 12
// CTAs 484.0, 40 at 12 CTAs 486.0, 48 at 12 CTAs 489.8, 64 at 11 CTAs 487.2, 96 at 10 CTAs
// 476.4; kSub 3 at 13 CTAs (78 registers) 468 with chunk 48, 478 with chunk 32.
#define NX_COMPOSITE_CHUNK 48
#endif
#ifndef NX_COMPOSITE_SUB
#define NX_COMPOSITE_SUB 4
#endif
constexpr int kChunk = NX_COMPOSITE_CHUNK;       // primitives staged per round (<= 256)
constexpr int kSub = NX_COMPOSITE_SUB;           // primitives pooled per B1/B2 round
constexpr int kPool = 32 * kSub;
constexpr int kRecPieces = REC_FIELDS * 8 / 16;  // 16-byte pieces of an fp64 record (10)
constexpr int kShPieces = NX_SH_VALUES * 4 / 16; // 16-byte pieces of the SH coefficients (12)
// Staged rows are padded by 16 bytes (208-byte stride): the B1 lanes of a warp read up
// to kSub different rows at once, and at the unpadded 192-byte stride rows 0 / 2 and
// 1 / 3 fall on the same banks (two-way conflicts on every record and SH load).
// Measured at config 2 (composite stage ms / frames/s): padded 1.036 / 488; no padding
// (12 CTAs / SM fit) 1.123 / 469; no record padding with kSub 3 at 12 CTAs 1.107 / 481;
// kSub 3 padded at 12 CTAs 1.055 / 486.
#ifndef NX_REC_PAD
#define NX_REC_PAD 2
#endif
#ifndef NX_SH_PAD
#define NX_SH_PAD 4
#endif
constexpr int kRecStride = REC_FIELDS + NX_REC_PAD;
constexpr int kShStride = NX_SH_VALUES + NX_SH_PAD;
static_assert(kWorkTile == 8, "warp blocks are 8x4 pixels");
#ifndef NX_NEAR_COUNTERS
#define NX_NEAR_COUNTERS 1
#endif
constexpr bool kNear = NX_NEAR_COUNTERS;  // near-threshold decision counters (FrameStatsD::near)
#ifndef NX_QUAD_CULL
#define NX_QUAD_CULL 1
#endif
constexpr bool kQuadCull = NX_QUAD_CULL;  // per-warp cull of the projected support (sel phase)
static_assert(kChunk <= 256 && kSub <= 8, "pool entries pack (lane, group slot) in 16 bits");

template <typename CT>  // colour type: float, or double for NX_PRECISION_F64
struct PoolEntry {         // one evaluated (pixel, primitive) pair
    double alpha;          // raw kernel alpha, < 0 for a miss
    double t;              // plane crossing
    CT rgb[3];             // primitive colour along the ray
    int32_t id;
    static constexpr bool kHasId = true;
    __device__ __forceinline__ void set_id(int32_t i) { id = i; }
};

// Certified mode: alpha from the SFU with its error bound (cert_alpha), 1 - alpha and
// the bounds travel with the entry so that B2 can certify T and the top-K order.
#ifndef NX_POOL_PACKED
#define NX_POOL_PACKED 1  // 32-byte certified entries: 18.4 KB of shared memory per CTA, 11 CTAs / SM
#endif
#if NX_POOL_PACKED
// 32 bytes: the two bounds as fp16 scaled by 2^20 and rounded up (an overflow reads as
// an infinite bound, i.e. a redo), no id: B2 recovers it from the lane's survivor mask
struct PoolEntryCert {
    static constexpr bool kHasId = false;
    double t;
    float alpha;  // clamped kernel alpha (< 0: miss)
    float oma;    // 1 - alpha
    __half2 eps2;
    float rgb[3];
    __device__ __forceinline__ void set_eps(float e, float eo) {
        eps2 = __halves2half2(__float2half_ru(e * 1048576.f), __float2half_ru(eo * 1048576.f));
    }
    __device__ __forceinline__ float eps() const { return __low2float(eps2) * 9.5367431640625e-07f; }
    __device__ __forceinline__ float eps_oma() const { return __high2float(eps2) * 9.5367431640625e-07f; }
    __device__ __forceinline__ void set_id(int32_t) {}
};
#else
struct PoolEntryCert {
    static constexpr bool kHasId = true;
    double t;
    float alpha;     // clamped kernel alpha (< 0: miss)
    float oma;       // 1 - alpha
    float eps_;      // relative error bound of alpha
    float eps_oma_;  // relative error bound of oma
    float rgb[3];
    int32_t id;
    __device__ __forceinline__ void set_eps(float e, float eo) {
        eps_ = e;
        eps_oma_ = eo;
    }
    __device__ __forceinline__ float eps() const { return eps_; }
    __device__ __forceinline__ float eps_oma() const { return eps_oma_; }
    __device__ __forceinline__ void set_id(int32_t i) { id = i; }
};
#endif

template <typename PE>
struct alignas(16) WarpStage {  // one warp's private staging
    double rec[kSub][kRecStride];    // exact records of the group's primitives
    float sh[kSub][kShStride];       // and their SH coefficients (fp32 colour path)
    uint8_t sel[kChunk];             // chunk slots whose pixel rect meets the warp's block
    uint32_t lmask[kChunk];          // and the lanes (pixels of the 8x4 block) inside that rect
    uint16_t q[kPool];
    PE res[kPool];
};

template <typename PE>
struct SmemLayout {
    float4 f[kChunk][4];
    int32_t id[kChunk];
    double dir[kThreads][3];
    float cdir[kWarps][4][3];  // the ray directions of each warp block's corner pixels
    WarpStage<PE> w[kWarps];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

// Primitive SH colour (eval_sh, sh.hpp:46-57) in fp32 from staged coefficients: the
// same operations, in the same order, as eval_sh_f32 (nx_composite.cuh).
// The coefficients are read as 16-byte vectors (12 loads instead of 48).
__device__ __forceinline__ void eval_sh_smem(const float* sh, float x, float y, float z, int degree, float* rgb) {
    const float4* s4 = reinterpret_cast<const float4*>(sh);
    const float4 v0 = s4[0];
    float a0 = 0.5f + 0.28209479177387814f * v0.x;
    float a1 = 0.5f + 0.28209479177387814f * v0.y;
    float a2 = 0.5f + 0.28209479177387814f * v0.z;
    if (degree >= 3) {
        float b[16];
        sh_basis_f32(x, y, z, b);
        float c[48];
        c[3] = v0.w;
#pragma unroll
        for (int q = 1; q < 12; ++q) {
            const float4 v = s4[q];
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
    rgb[0] = fmaxf(a0, 0.f);
    rgb[1] = fmaxf(a1, 0.f);
    rgb[2] = fmaxf(a2, 0.f);
}

template <int K, bool kDebug, typename CT, bool kCert>
#ifndef NX_COMPOSITE_MINB
#define NX_COMPOSITE_MINB 12  // certified pass, measured (packed entries, chunk 64): 10 1.076 ms, 11 1.059, 12 1.061; chunk 48: 12
#endif
// (the exact-path variants keep 10: their larger pool entries fit 10 CTAs of shared memory anyway)
__global__ void __launch_bounds__(kThreads, kCert ? NX_COMPOSITE_MINB : 10) composite_kernel(const CompositeArgs a) {
    constexpr int KK = K > 0 ? K : 1;
    constexpr bool kKeepRgb = K <= 4;  // top-K slots remember their colour (else re-evaluated at the end)
    constexpr int KR = kKeepRgb ? KK : 1;
    constexpr bool kF64 = sizeof(CT) == 8;  // NX_PRECISION_F64: fp64 SH colour from the fp64 copy
    static_assert(!(kCert && kF64), "the certified fp32 alpha serves the fp32-colour path");
    using PE = std::conditional_t<kCert, PoolEntryCert, PoolEntry<CT>>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SmemLayout<PE>& sm = *reinterpret_cast<SmemLayout<PE>*>(smem_raw);

    const int t = blockIdx.x;
    const int tx = t % a.fb.tiles_x, ty = t / a.fb.tiles_x;
    const int list_begin = a.tile_offsets[t], list_end = a.tile_offsets[t + 1];
    const int W = a.cam.W, H = a.cam.H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpStage<PE>& ws = sm.w[warp];
    const double near_eps = a.st.near_eps, alpha_max = a.st.alpha_max, min_T = a.st.min_transmittance;
    const float near_eps_f = static_cast<float>(near_eps);

    // warp w owns pixel rows 4w..4w+3 of the 8x8 tile
    const int px = tx * kWorkTile + (lane & 7), py = ty * kWorkTile + warp * 4 + (lane >> 3);
    const bool in_img = px < W && py < H;
    const int wx0 = __reduce_min_sync(0xffffffffu, in_img ? px : 0x7fffffff);
    const int wx1 = __reduce_max_sync(0xffffffffu, in_img ? px : -1);
    const int wy0 = __reduce_min_sync(0xffffffffu, in_img ? py : 0x7fffffff);
    const int wy1 = __reduce_max_sync(0xffffffffu, in_img ? py : -1);
    double dir[3] = {0.0, 0.0, 1.0};
    if (in_img) pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
    sm.dir[threadIdx.x][0] = dir[0];
    sm.dir[threadIdx.x][1] = dir[1];
    sm.dir[threadIdx.x][2] = dir[2];
    // the warp block's corner pixels (lanes 0, 7, 24, 31): the per-warp cull of the
    // projected support below needs every corner in the image
    const uint32_t in_mask = __ballot_sync(0xffffffffu, in_img);
    constexpr uint32_t kCorners = (1u << 0) | (1u << 7) | (1u << 24) | (1u << 31);
    const bool quad_ok = kQuadCull && (in_mask & kCorners) == kCorners;
    {
        const int ci = lane == 0 ? 0 : lane == 7 ? 1 : lane == 24 ? 2 : lane == 31 ? 3 : -1;
        if (ci >= 0) {
            sm.cdir[warp][ci][0] = static_cast<float>(dir[0]);
            sm.cdir[warp][ci][1] = static_cast<float>(dir[1]);
            sm.cdir[warp][ci][2] = static_cast<float>(dir[2]);
        }
    }
    const float dfx = static_cast<float>(dir[0]), dfy = static_cast<float>(dir[1]), dfz = static_cast<float>(dir[2]);

    // March precision: fp64 on the exact path; the certified pass marches in fp32 (its
    // alphas are fp32 already) and folds each fp32 rounding of T and of a weight into
    // the tracked bounds (kCertRound), so every decision it takes stays certified.
#ifndef NX_CERT_F32_MARCH
#define NX_CERT_F32_MARCH 1
#endif
    using TT = std::conditional_t<kCert && NX_CERT_F32_MARCH, float, double>;
    constexpr float kCertRound = 1.2e-7f;  // > 2^-23: one fp32 rounding, with slack
    TT T = 1.0;
    TT acc[3] = {0.0, 0.0, 0.0};
    int32_t k_id[KK];
    TT k_w[KK];
    double k_t[KK];
    CT k_rgb[KR][3];
#pragma unroll
    for (int s = 0; s < KK; ++s) {
        k_id[s] = -1;
        k_w[s] = 0.0;
        k_t[s] = 0.0;
    }
#pragma unroll
    for (int s = 0; s < KR; ++s) k_rgb[s][0] = k_rgb[s][1] = k_rgb[s][2] = CT(0);
    int k_size = 0;
    bool active = in_img;
    // near-threshold decisions of this pixel (kNear), packed: alpha | T << 10 | top-K << 20
    // (per-pixel counts stay far below 1024)
    uint32_t n_near = 0;
    float E_T = 0.f;        // certified mode: relative error bound of T
    // and, per top-K slot, the alpha bound and E_T when it was inserted: two weights'
    // ratio carries only their alphas' errors and the 1 - alpha factors between them
    float k_ea[KK], k_et[KK];
    bool unsure = false;    // a decision this pass could not certify: the tile is redone exactly
#pragma unroll
    for (int s = 0; s < KK; ++s) k_ea[s] = k_et[s] = 0.f;
    int dbg_n = 0;
    const bool dbg_row = kDebug && in_img && py >= a.dbg_y0 && py < a.dbg_y1;
    const int64_t dbg_q = kDebug ? (static_cast<int64_t>(py - a.dbg_y0) * W + px) : 0;

    for (int cb = list_begin; cb < list_end; cb += kChunk) {
        const int cn = min(kChunk, list_end - cb);
        __syncthreads();
        // the chunk's fp32 prefilter records (gathered by id) into shared memory with
        // asynchronous 16-byte copies (cp.async: global -> shared without a register trip)
        for (int e = threadIdx.x; e < cn * 4; e += kThreads) {
            const int j = e >> 2, q = e & 3;
            const int32_t id = __ldg(a.list_ids + cb + j);
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&sm.f[j][q]));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(a.recf + static_cast<int64_t>(id) * 4 + q)
                         : "memory");
            if (q == 0) sm.id[j] = id;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (__any_sync(0xffffffffu, active)) {
            // ---- 0. the chunk's primitives whose pixel rect meets this warp's block, in order
            int nsel = 0;
            const int bx0 = tx * kWorkTile, by0 = ty * kWorkTile + warp * 4;  // the warp block's origin
            for (int b0 = 0; b0 < cn; b0 += 32) {
                const int b = b0 + lane;
                bool ov = false;
                uint32_t lm = 0;
                if (b < cn) {
                    const float4 f3 = sm.f[b][3];
                    const int rx = __float_as_int(f3.z), ry = __float_as_int(f3.w);
                    ov = !((rx >> 16) < wx0 || (rx & 0xffff) > wx1 || (ry >> 16) < wy0 || (ry & 0xffff) > wy1);
                    if (ov && quad_ok) {
                        // The plane offsets (u, v) of the block's pixel rays are a projective
                        // image of the pixel rectangle, so they lie in the quadrilateral of
                        // the corner rays' offsets when all four cross the plane on one side:
                        // if that quadrilateral (enlarged by the prefilter's slack) misses the
                        // support box, every pixel of the block misses.
                        const float4 f0 = sm.f[b][0], f1 = sm.f[b][1], f2 = sm.f[b][2];
                        float umin = 3e38f, umax = -3e38f, vmin = 3e38f, vmax = -3e38f, su = 0.f, sv = 0.f;
                        bool valid = true;
                        float sgn = 0.f;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float dx = sm.cdir[warp][c][0], dy = sm.cdir[warp][c][1], dz = sm.cdir[warp][c][2];
                            const float den = dx * f0.x + dy * f0.y + dz * f0.z;
                            valid &= fabsf(den) >= 1e-2f && (c == 0 || den * sgn > 0.f);
                            sgn = den;
                            const float ta = __fdividef(f0.w, den);
                            const float ta1 = ta * (dx * f1.x + dy * f1.y + dz * f1.z);
                            const float ta2 = ta * (dx * f2.x + dy * f2.y + dz * f2.z);
                            const float u = ta1 - f1.w, v = ta2 - f2.w;
                            umin = fminf(umin, u);
                            umax = fmaxf(umax, u);
                            vmin = fminf(vmin, v);
                            vmax = fmaxf(vmax, v);
                            su = fmaxf(su, 1e-4f * (fabsf(ta1) + fabsf(ta) + fabsf(f1.w)) + 1e-7f);
                            sv = fmaxf(sv, 1e-4f * (fabsf(ta2) + fabsf(ta) + fabsf(f2.w)) + 1e-7f);
                        }
                        if (valid && (umin > f3.x + su || umax < -f3.x - su || vmin > f3.y + sv || vmax < -f3.y - sv))
                            ov = false;
                    }
                    if (ov) {  // lane l = pixel (bx0 + l % 8, by0 + l / 8): the rect's columns x its rows
                        const int cx0 = max((rx & 0xffff) - bx0, 0), cx1 = min((rx >> 16) - bx0, 7);
                        const int ry0 = max((ry & 0xffff) - by0, 0), ry1 = min((ry >> 16) - by0, 3);
                        const uint32_t cols = (0xffu >> (7 - cx1)) & (0xffu << cx0);
                        const uint32_t rows = (0xffffffffu >> (8 * (3 - ry1))) & (0xffffffffu << (8 * ry0));
                        lm = (cols * 0x01010101u) & rows;
                    }
                }
                const uint32_t m = __ballot_sync(0xffffffffu, ov);
                if (ov) {
                    const int slot = nsel + __popc(m & ((1u << lane) - 1u));
                    ws.sel[slot] = static_cast<uint8_t>(b);
                    ws.lmask[slot] = lm;
                }
                nsel += __popc(m);
            }
            __syncwarp();
            for (int g0 = 0; g0 < nsel; g0 += kSub) {
                const int gn = min(kSub, nsel - g0);
                // ---- S. stage the group's exact records + SH coefficients (asynchronous)
                constexpr int kPieces = kRecPieces + (kF64 ? 0 : kShPieces);
                for (int e = lane; e < gn * kPieces; e += 32) {
                    const int b = e / kPieces, pc = e - b * kPieces;
                    const int64_t id = sm.id[ws.sel[g0 + b]];
                    if (pc < kRecPieces)
                        cp_async16(reinterpret_cast<float4*>(ws.rec[b]) + pc,
                                   reinterpret_cast<const float4*>(a.rec + id * REC_FIELDS) + pc);
                    else
                        cp_async16(reinterpret_cast<float4*>(ws.sh[b]) + (pc - kRecPieces),
                                   reinterpret_cast<const float4*>(a.sh + id * NX_SH_VALUES) + (pc - kRecPieces));
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                // ---- A. per-pixel rect test + fp32 prefilter of the group
                uint32_t mask = 0;
                if (active) {
#pragma unroll 4
                    for (int b = 0; b < gn; ++b) {
                        const int j = ws.sel[g0 + b];
                        if (((ws.lmask[g0 + b] >> lane) & 1u) && prefilter(&sm.f[j][0], dfx, dfy, dfz, near_eps_f))
                            mask |= 1u << b;
                    }
                }
                // warp-wide pool: exclusive offsets of each lane's survivors
                const int cnt = __popc(mask);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int off = incl - cnt;
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (total == 0) {
                    asm volatile("cp.async.wait_all;" ::: "memory");  // the staging is reused next group
                    __syncwarp();
                    continue;
                }
                {
                    uint32_t m = mask;
                    int k = off;
                    while (m) {
                        const int b = __ffs(m) - 1;
                        m &= m - 1;
                        ws.q[k++] = static_cast<uint16_t>((lane << 8) | b);
                    }
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                // ---- B1. exact fp64 evaluation of the pooled pairs, all lanes busy
                for (int e = lane; e < total; e += 32) {
                    const int ent = ws.q[e];
                    const int owner = ent >> 8, b = ent & 0xf;
                    const double* dd = sm.dir[warp * 32 + owner];
                    const double d0 = dd[0], d1 = dd[1], d2 = dd[2];
                    const double* r = ws.rec[b];
                    PE res;
                    res.alpha = -1.0;
                    res.t = 0.0;
                    const int32_t pid = sm.id[ws.sel[g0 + b]];
                    res.set_id(pid);
                    if constexpr (kCert) {
                        // intersect (intersect.hpp:23-42) in fp64 up to the plane offsets, then the
                        // kernel value on the SFU with its error bound; decisions the bound does
                        // not clear take the exact fp64 routine
                        const double denom = d0 * r[REC_NX] + d1 * r[REC_NY] + d2 * r[REC_NZ];
                        if (fabs(denom) >= kMinNormalDot) {
                            const double tt = r[REC_NUM] / denom;
                            if (tt > near_eps) {
                                const double e0 = (a.cam.o[0] + tt * d0) - r[REC_MUX];
                                const double e1 = (a.cam.o[1] + tt * d1) - r[REC_MUY];
                                const double e2 = (a.cam.o[2] + tt * d2) - r[REC_MUZ];
                                const double du = e0 * r[REC_V1X] + e1 * r[REC_V1Y] + e2 * r[REC_V1Z];
                                const double dv = e0 * r[REC_V2X] + e1 * r[REC_V2Y] + e2 * r[REC_V2Z];
                                if (fabs(du) <= r[REC_ULIM] && fabs(dv) <= r[REC_VLIM]) {
                                    const CertAlpha c = cert_alpha(
                                        static_cast<float>(du) * static_cast<float>(r[REC_RSX]),
                                        static_cast<float>(dv) * static_cast<float>(r[REC_RSY]),
                                        static_cast<float>(2.0 * r[REC_GX]), static_cast<float>(2.0 * r[REC_GY]),
                                        static_cast<float>(r[REC_OP]), static_cast<float>(r[REC_OM]));
                                    const double al = c.alpha, lo = al * (1.0 - c.eps), hi = al * (1.0 + c.eps);
                                    const bool sure = (lo >= kAlphaMin || hi < kAlphaMin) &&
                                                      (lo > alpha_max || hi <= alpha_max);
                                    if (sure) {
                                        if (lo >= kAlphaMin) {
                                            res.t = tt;
                                            if (lo > alpha_max) {  // clamped: alpha_max exactly
                                                res.alpha = static_cast<float>(alpha_max);
                                                res.oma = static_cast<float>(1.0 - alpha_max);
                                                res.set_eps(6e-8f, 6e-8f);
                                            } else {
                                                res.alpha = c.alpha;
                                                res.oma = c.oma;
                                                res.set_eps(c.eps, c.eps_oma);
                                            }
                                        }
                                    } else {  // the exact routine decides (rare)
                                        const HitTerms h =
                                            exact_hit(r, d0, d1, d2, a.cam.o[0], a.cam.o[1], a.cam.o[2], near_eps);
                                        if (kNear) n_near += h.near ? 1u : 0u;
                                        if (h.alpha >= 0.0) {
                                            const double ac = alpha_max < h.alpha ? alpha_max : h.alpha;
                                            res.t = h.t;
                                            res.alpha = static_cast<float>(ac);
                                            res.oma = static_cast<float>(1.0 - ac);
                                            res.set_eps(1.2e-7f, 1.2e-7f);
                                        }
                                    }
                                    if (res.alpha >= 0.f)
                                        eval_sh_smem(ws.sh[b], static_cast<float>(d0), static_cast<float>(d1),
                                                     static_cast<float>(d2), a.sh_degree, res.rgb);
                                }
                            }
                        }
                    } else {
                        // intersect (intersect.hpp:23-42) + eval_kernel (kernel.hpp:16-30)
                        const HitTerms h = exact_hit(r, d0, d1, d2, a.cam.o[0], a.cam.o[1], a.cam.o[2], near_eps);
                        if (kNear) n_near += h.near ? 1u : 0u;
                        if (h.alpha >= 0.0) {
                            res.alpha = h.alpha;
                            res.t = h.t;
                            if constexpr (kF64) {
                                const double dd3[3] = {d0, d1, d2};
                                eval_sh_f64(a.sh64 + static_cast<int64_t>(pid) * NX_SH_VALUES, dd3, a.sh_degree,
                                            res.rgb);
                            } else {
                                eval_sh_smem(ws.sh[b], static_cast<float>(d0), static_cast<float>(d1),
                                             static_cast<float>(d2), a.sh_degree, res.rgb);
                            }
                        }
                    }
                    ws.res[e] = res;
                }
                __syncwarp();
                // ---- B2. per-pixel compositing of this lane's hits, in list order (renderer.cpp:144-153)
                uint32_t mrem = mask;  // this lane's survivors in group order (ids of packed entries)
                for (int k = off; k < off + cnt && active; ++k) {
                    const PE& res = ws.res[k];
                    const int bk = __ffs(mrem) - 1;
                    mrem &= mrem - 1;
                    if (res.alpha < 0.0) continue;
                    int32_t id;
                    if constexpr (PE::kHasId) id = res.id;
                    else id = sm.id[ws.sel[g0 + bk]];
                    // (certified entries arrive clamped)
                    const TT alpha = kCert ? static_cast<TT>(res.alpha)
                                           : static_cast<TT>(alpha_max < res.alpha ? alpha_max : static_cast<double>(res.alpha));
                    const TT wgt = alpha * T;
                    float eps_a = 0.f;  // certified mode: alpha's relative error bound
                    if constexpr (kCert) eps_a = res.eps();
                    acc[0] += wgt * res.rgb[0];
                    acc[1] += wgt * res.rgb[1];
                    acc[2] += wgt * res.rgb[2];
                    if (K > 0) {
                        // TopKBuffer::insert (framebuffers.hpp:33-48) with the slots kept in the
                        // finalize order (weight desc, arrival asc; framebuffers.hpp:51-56): the
                        // last-ranked incumbent the reference replaces (smallest weight, latest
                        // arrival among ties) is then always the last slot, and finalize has
                        // nothing left to sort. A new entry arrives last, so among equal weights it
                        // ranks behind every incumbent: it moves up only past strictly smaller ones.
                        // Certified mode: every comparison taken is checked against the weights'
                        // error bounds (the ratio of two weights carries their alphas' errors and
                        // the 1 - alpha factors between their insertions).
                        int pos = -1;
                        if (k_size < K) {
                            pos = k_size++;
                        } else {
                            const TT wm = k_w[KK - 1];
                            if (kCert && fabs(wgt - wm) <= (eps_a + k_ea[KK - 1] + (E_T - k_et[KK - 1]) + 2.f * kCertRound) *
                                                               fmax(wgt, wm))
                                unsure = true;
                            if (kNear && !kCert) n_near += (wgt != wm) & (fabs(wgt - wm) <= kNearRel * wm) ? (1u << 20) : 0u;
                            if (wgt > wm) pos = KK - 1;
                        }
#pragma unroll
                        for (int s = 0; s < KK; ++s)
                            if (s == pos) {
                                k_id[s] = id;
                                k_w[s] = wgt;
                                k_t[s] = res.t;
                                k_ea[s] = eps_a;
                                k_et[s] = E_T;
                                if (kKeepRgb) {
                                    k_rgb[s % KR][0] = res.rgb[0];
                                    k_rgb[s % KR][1] = res.rgb[1];
                                    k_rgb[s % KR][2] = res.rgb[2];
                                }
                            }
#pragma unroll
                        for (int s = KK - 1; s >= 1; --s)
                            if (s == pos) {
                                const TT wp = k_w[s - 1];
                                if (kCert && fabs(wgt - wp) <= (eps_a + k_ea[s - 1] + (E_T - k_et[s - 1]) + 2.f * kCertRound) *
                                                                   fmax(wgt, wp))
                                    unsure = true;
                                if (kNear && !kCert)
                                    n_near += (wgt != wp) & (fabs(wgt - wp) <= kNearRel * wp) ? (1u << 20) : 0u;
                                if (wgt > wp) {
                                    pos = s - 1;
                                    k_id[s] = k_id[s - 1];
                                    k_w[s] = k_w[s - 1];
                                    k_t[s] = k_t[s - 1];
                                    k_ea[s] = k_ea[s - 1];
                                    k_et[s] = k_et[s - 1];
                                    k_id[s - 1] = id;
                                    k_w[s - 1] = wgt;
                                    k_t[s - 1] = res.t;
                                    k_ea[s - 1] = eps_a;
                                    k_et[s - 1] = E_T;
                                    if (kKeepRgb) {
#pragma unroll
                                        for (int c = 0; c < 3; ++c) {
                                            k_rgb[s % KR][c] = k_rgb[(s - 1) % KR][c];
                                            k_rgb[(s - 1) % KR][c] = res.rgb[c];
                                        }
                                    }
                                }
                            }
                    }
                    if (kDebug && dbg_row) {
                        if (dbg_n < a.dbg_max) a.dbg_hits[dbg_q * a.dbg_max + dbg_n] = id;
                        ++dbg_n;
                    }
                    if constexpr (kCert) {  // T *= 1 - alpha with 1 - alpha from the entry (no cancellation)
                        T *= res.oma;
                        E_T += res.eps_oma() + kCertRound;
                        // T vs min_T uncertain (fp32 min_T and the subtraction: one more rounding each)
                        if (fabs(T - static_cast<TT>(min_T)) <= (E_T + 2.f * kCertRound) * fmax(T, static_cast<TT>(min_T)))
                            unsure = true;
                    } else {
                        T *= 1.0 - alpha;
                    }
                    if (static_cast<double>(T) < min_T) active = false;
                    // (certified pass: uncertain T / top-K decisions are redone exactly and counted there)
                    if (kNear && !kCert) n_near += fabs(T - min_T) <= kNearRel * min_T ? (1u << 10) : 0u;
                }
                __syncwarp();
            }
        }
        if (cb + kChunk < list_end && !__syncthreads_or(active)) break;
    }

    if (in_img) {
        const int64_t pix = static_cast<int64_t>(py) * W + px;
        a.fb.residual[pix] = static_cast<float>(T);
        if (a.fb.residual64) a.fb.residual64[pix] = T;
        acc[0] += T * static_cast<TT>(a.st.background[0]);
        acc[1] += T * static_cast<TT>(a.st.background[1]);
        acc[2] += T * static_cast<TT>(a.st.background[2]);
        if (K > 0) {
            // finalize (framebuffers.hpp:51-56): the slots are already in rank order; slots >= size
            // keep their sentinels.
            // write slots; subtract the buffered primitives' own colours (renderer.cpp:157-164)
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int64_t sl = pix * K + j;
                a.fb.ids[sl] = k_id[j];
                a.fb.depths[sl] = k_t[j];
                a.fb.weights[sl] = k_w[j];
                if (j < k_size) {
                    CT col[3];
                    if (kKeepRgb) {
                        col[0] = k_rgb[j % KR][0];
                        col[1] = k_rgb[j % KR][1];
                        col[2] = k_rgb[j % KR][2];
                    } else if constexpr (kF64) {
                        eval_sh_f64(a.sh64 + static_cast<int64_t>(k_id[j]) * NX_SH_VALUES, dir, a.sh_degree, col);
                    } else {
                        eval_sh_f32(a.sh + static_cast<int64_t>(k_id[j]) * NX_SH_VALUES, dfx, dfy, dfz, a.sh_degree,
                                    col);
                    }
                    acc[0] -= k_w[j] * col[0];
                    acc[1] -= k_w[j] * col[1];
                    acc[2] -= k_w[j] * col[2];
                }
            }
        }
        a.fb.base[pix * 3 + 0] = static_cast<float>(acc[0]);
        a.fb.base[pix * 3 + 1] = static_cast<float>(acc[1]);
        a.fb.base[pix * 3 + 2] = static_cast<float>(acc[2]);
        if (a.fb.base64) {  // fp64 base kept for render_backward (nx_frame_set_backward)
            a.fb.base64[pix * 3 + 0] = acc[0];
            a.fb.base64[pix * 3 + 1] = acc[1];
            a.fb.base64[pix * 3 + 2] = acc[2];
        }
        if (kDebug && dbg_row) a.dbg_counts[dbg_q] = dbg_n;
        if (kCert && (unsure || a.redo_all)) {  // a decision the bounds did not clear: redone exactly
            const int slot = atomicAdd(a.redo, 1);
            a.redo[1 + slot] = static_cast<int32_t>(pix);
        }
    }
    if (kNear && n_near) {
        if (n_near & 1023u) atomicAdd(&a.stats->near[NEAR_ALPHA], static_cast<unsigned long long>(n_near & 1023u));
        if ((n_near >> 10) & 1023u)
            atomicAdd(&a.stats->near[NEAR_TRANSMITTANCE], static_cast<unsigned long long>((n_near >> 10) & 1023u));
        if (n_near >> 20) atomicAdd(&a.stats->near[NEAR_TOPK], static_cast<unsigned long long>(n_near >> 20));
    }
}


// Exact redo of the pixels the certified pass could not certify: one warp per pixel. The
// lanes evaluate 32 list entries at a time (pixel rect test + the exact fp64 intersect /
// eval_kernel, exact_hit, + SH colour), the hits are packed in list order, and lane 0
// composites them sequentially with the exact pass's arithmetic (renderer.cpp:144-164),
// so a redone pixel carries the exact composite's bits.
template <int K, bool kDebug>
__global__ void __launch_bounds__(256) redo_pixels_kernel(const CompositeArgs a) {
    constexpr int KK = K > 0 ? K : 1;
    // One CTA per redo pixel: the 256 threads intersect 256 list entries at a time (the
    // exact fp64 hit, SH for the hits), the hits are compacted in list order into shared
    // memory and thread 0 marches them exactly like the collection pass. The per-pixel
    // chain is one L2 round trip per 256 entries instead of per 32 (a few hundred redo
    // pixels per frame, each a dense tile's list of ~1000 entries).
    struct Hits {
        double alpha[256], t[256];
        float rgb[256][3];
        int32_t id[256];
    };
    __shared__ Hits h;
    __shared__ int s_wc[8];
    __shared__ int s_active;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = *a.redo;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.stats->redo_tiles = static_cast<unsigned long long>(n);
    const int W = a.cam.W;
    const double near_eps = a.st.near_eps, alpha_max = a.st.alpha_max, min_T = a.st.min_transmittance;
    const double2* rec2 = reinterpret_cast<const double2*>(a.rec);
    uint32_t n_near = 0;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t pix = a.redo[1 + i];
        const int px = static_cast<int>(pix % W), py = static_cast<int>(pix / W);
        const int t = (py / kWorkTile) * a.fb.tiles_x + px / kWorkTile;
        const int list_begin = a.tile_offsets[t], list_end = a.tile_offsets[t + 1];
        double dir[3];
        pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
        const float dfx = static_cast<float>(dir[0]), dfy = static_cast<float>(dir[1]), dfz = static_cast<float>(dir[2]);
        double T = 1.0, acc[3] = {0.0, 0.0, 0.0};
        int32_t k_id[KK];
        double k_w[KK], k_t[KK];
        uint32_t k_seq[KK];
        float k_rgb[KK][3];
        for (int s = 0; s < KK; ++s) {
            k_id[s] = -1;
            k_w[s] = 0.0;
            k_t[s] = 0.0;
            k_seq[s] = 0;
            k_rgb[s][0] = k_rgb[s][1] = k_rgb[s][2] = 0.f;
        }
        int k_size = 0, dbg_n = 0;
        uint32_t counter = 0;
        bool active = true;
        const bool dbg_row = kDebug && py >= a.dbg_y0 && py < a.dbg_y1;
        const int64_t dbg_q = kDebug ? (static_cast<int64_t>(py - a.dbg_y0) * W + px) : 0;
        for (int cb = list_begin; cb < list_end && active; cb += 256) {
            const int e = cb + static_cast<int>(threadIdx.x);
            bool hit = false;
            double al = 0.0, tt = 0.0;
            float rgb[3] = {0.f, 0.f, 0.f};
            int32_t id = -1;
            if (e < list_end) {
                id = a.list_ids[e];
                const float4 f3 = __ldg(a.recf + static_cast<int64_t>(id) * 4 + 3);
                const int rx = __float_as_int(f3.z), ry = __float_as_int(f3.w);
                if (px >= (rx & 0xffff) && px <= (rx >> 16) && py >= (ry & 0xffff) && py <= (ry >> 16)) {
                    double r[REC_FIELDS];
#pragma unroll
                    for (int q = 0; q < REC_FIELDS / 2; ++q) {
                        const double2 v = __ldg(rec2 + static_cast<int64_t>(id) * (REC_FIELDS / 2) + q);
                        r[2 * q] = v.x;
                        r[2 * q + 1] = v.y;
                    }
                    const HitTerms ht = exact_hit(r, dir[0], dir[1], dir[2], a.cam.o[0], a.cam.o[1], a.cam.o[2],
                                                  near_eps);
                    n_near += ht.near ? 1u : 0u;
                    if (ht.alpha >= 0.0) {
                        hit = true;
                        al = ht.alpha;
                        tt = ht.t;
                        eval_sh_f32(a.sh + static_cast<int64_t>(id) * NX_SH_VALUES, dfx, dfy, dfz, a.sh_degree, rgb);
                    }
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            if (lane == 0) s_wc[warp] = __popc(m);
            __syncthreads();
            int off = 0, nh = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const int c = s_wc[w];
                off += w < warp ? c : 0;
                nh += c;
            }
            if (hit) {
                const int k = off + __popc(m & ((1u << lane) - 1u));
                h.alpha[k] = al;
                h.t[k] = tt;
                h.rgb[k][0] = rgb[0];
                h.rgb[k][1] = rgb[1];
                h.rgb[k][2] = rgb[2];
                h.id[k] = id;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int k = 0; k < nh && active; ++k) {
                    const double alpha = alpha_max < h.alpha[k] ? alpha_max : h.alpha[k];
                    const double wgt = alpha * T;
                    acc[0] += wgt * h.rgb[k][0];
                    acc[1] += wgt * h.rgb[k][1];
                    acc[2] += wgt * h.rgb[k][2];
                    if (K > 0) {  // TopKBuffer::insert (framebuffers.hpp:33-48)
                        const uint32_t seq = counter++;
                        int slot = -1;
                        if (k_size < K) {
                            slot = k_size++;
                        } else {
                            int mi = 0;
                            double wm = k_w[0];
                            uint32_t qm = k_seq[0];
                            for (int s = 1; s < KK; ++s)
                                if (k_w[s] < wm || (k_w[s] == wm && k_seq[s] > qm)) {
                                    mi = s;
                                    wm = k_w[s];
                                    qm = k_seq[s];
                                }
                            if (wgt > wm) slot = mi;
                            n_near += (wgt != wm) & (fabs(wgt - wm) <= kNearRel * wm) ? (1u << 20) : 0u;
                        }
                        if (slot >= 0) {
                            k_id[slot] = h.id[k];
                            k_w[slot] = wgt;
                            k_t[slot] = h.t[k];
                            k_seq[slot] = seq;
                            k_rgb[slot][0] = h.rgb[k][0];
                            k_rgb[slot][1] = h.rgb[k][1];
                            k_rgb[slot][2] = h.rgb[k][2];
                        }
                    }
                    if (kDebug && dbg_row) {
                        if (dbg_n < a.dbg_max) a.dbg_hits[dbg_q * a.dbg_max + dbg_n] = h.id[k];
                        ++dbg_n;
                    }
                    T *= 1.0 - alpha;
                    if (T < min_T) active = false;
                    n_near += fabs(T - min_T) <= kNearRel * min_T ? (1u << 10) : 0u;
                }
                s_active = active;
            }
            __syncthreads();
            active = s_active;
        }
        if (threadIdx.x == 0) {  // the exact pass's epilogue (renderer.cpp:155-164, framebuffers.hpp:51-56)
            a.fb.residual[pix] = static_cast<float>(T);
            if (a.fb.residual64) a.fb.residual64[pix] = T;
            acc[0] += T * a.st.background[0];
            acc[1] += T * a.st.background[1];
            acc[2] += T * a.st.background[2];
            if (K > 0) {
                for (int ii = 0; ii < K; ++ii)
                    for (int j = 0; j + 1 < K - ii; ++j) {
                        if (j + 1 < k_size && k_w[j + 1] != k_w[j] && fabs(k_w[j + 1] - k_w[j]) <= kNearRel * k_w[j])
                            n_near += 1u << 20;
                        const bool swap = (j + 1 < k_size) &&
                                          (k_w[j + 1] > k_w[j] || (k_w[j + 1] == k_w[j] && k_seq[j + 1] < k_seq[j]));
                        if (swap) {
                            const int32_t ti = k_id[j];
                            k_id[j] = k_id[j + 1];
                            k_id[j + 1] = ti;
                            const double tw = k_w[j];
                            k_w[j] = k_w[j + 1];
                            k_w[j + 1] = tw;
                            const double td = k_t[j];
                            k_t[j] = k_t[j + 1];
                            k_t[j + 1] = td;
                            const uint32_t ts = k_seq[j];
                            k_seq[j] = k_seq[j + 1];
                            k_seq[j + 1] = ts;
                            for (int c = 0; c < 3; ++c) {
                                const float tc = k_rgb[j][c];
                                k_rgb[j][c] = k_rgb[j + 1][c];
                                k_rgb[j + 1][c] = tc;
                            }
                        }
                    }
                for (int j = 0; j < K; ++j) {
                    const int64_t sl = pix * K + j;
                    a.fb.ids[sl] = k_id[j];
                    a.fb.depths[sl] = k_t[j];
                    a.fb.weights[sl] = k_w[j];
                    if (j < k_size) {
                        acc[0] -= k_w[j] * k_rgb[j][0];
                        acc[1] -= k_w[j] * k_rgb[j][1];
                        acc[2] -= k_w[j] * k_rgb[j][2];
                    }
                }
            }
            a.fb.base[pix * 3 + 0] = static_cast<float>(acc[0]);
            a.fb.base[pix * 3 + 1] = static_cast<float>(acc[1]);
            a.fb.base[pix * 3 + 2] = static_cast<float>(acc[2]);
            if (a.fb.base64) {
                a.fb.base64[pix * 3 + 0] = acc[0];
                a.fb.base64[pix * 3 + 1] = acc[1];
                a.fb.base64[pix * 3 + 2] = acc[2];
            }
            if (kDebug && dbg_row) {
                a.dbg_counts[dbg_q] = dbg_n;
                for (int ii = dbg_n; ii < a.dbg_max; ++ii) a.dbg_hits[dbg_q * a.dbg_max + ii] = -1;
            }
        }
        __syncthreads();
    }
    if (kNear && n_near) {
        if (n_near & 1023u) atomicAdd(&a.stats->near[NEAR_ALPHA], static_cast<unsigned long long>(n_near & 1023u));
        if ((n_near >> 10) & 1023u)
            atomicAdd(&a.stats->near[NEAR_TRANSMITTANCE], static_cast<unsigned long long>((n_near >> 10) & 1023u));
        if (n_near >> 20) atomicAdd(&a.stats->near[NEAR_TOPK], static_cast<unsigned long long>(n_near >> 20));
    }
}

template <int K, bool kDebug, typename CT, bool kCert>
void launch_variant(const CompositeArgs& a, unsigned grid, cudaStream_t s) {
    using PE = std::conditional_t<kCert, PoolEntryCert, PoolEntry<CT>>;
    const size_t smem = sizeof(SmemLayout<PE>);
    cudaFuncSetAttribute(composite_kernel<K, kDebug, CT, kCert>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    composite_kernel<K, kDebug, CT, kCert><<<grid, kThreads, smem, s>>>(a);
}

template <int K, bool kDebug>
void launch_one(const CompositeArgs& a, unsigned grid, cudaStream_t s) {
    if (a.sh64) {
        launch_variant<K, kDebug, double, false>(a, grid, s);
    } else if (a.certified && a.redo) {
        launch_variant<K, kDebug, float, true>(a, grid, s);  // certified pass, uncertain pixels -> redo
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H;
        const unsigned rgrid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(npix, sms * 4)));
        count_launch();
        redo_pixels_kernel<K, kDebug><<<rgrid, 256, 0, s>>>(a);  // the exact redo of those pixels
    } else {
        launch_variant<K, kDebug, float, false>(a, grid, s);
    }
}

template <bool kDebug>
void launch_k(const CompositeArgs& a, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(a.fb.tiles_x) * a.fb.tiles_y;
    if (grid == 0) return;
    switch (a.fb.K) {
        case 0: launch_one<0, kDebug>(a, grid, s); break;
        case 1: launch_one<1, kDebug>(a, grid, s); break;
        case 2: launch_one<2, kDebug>(a, grid, s); break;
        case 3: launch_one<3, kDebug>(a, grid, s); break;
        case 4: launch_one<4, kDebug>(a, grid, s); break;
        case 5: launch_one<5, kDebug>(a, grid, s); break;
        case 6: launch_one<6, kDebug>(a, grid, s); break;
        case 7: launch_one<7, kDebug>(a, grid, s); break;
        default: launch_one<8, kDebug>(a, grid, s); break;
    }
}

}  // namespace

void launch_composite(const CompositeArgs& a, cudaStream_t s) {
    count_launch();
    if (a.dbg_hits) launch_k<true>(a, s);
    else launch_k<false>(a, s);
}

}  // namespace nx
