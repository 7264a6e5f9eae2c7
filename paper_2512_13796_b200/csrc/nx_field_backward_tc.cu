// Field branch of render_backward, tensor-core variant for the reference field
// shape (16 levels x 2 features -> 32 -> 64 -> 64 -> 48): field_backward_batch
// (texture_field.cpp:77-146) over the buffered slots in three kernels, so that the
// latency-bound hash-grid gathers / scatters run at full occupancy and the MLP runs
// on tcgen05 with its weight gradients accumulated in TMEM:
//
//   G  features   one thread per slot: grid_lookup (hash_grid.cpp:26-83) at the
//                 query (x = o + t d, build_queries renderer.cpp:177-203) -> F[32]
//   M  mlp        persistent, one 128-slot tile per step, one thread per row:
//                 forward  H1 = relu(F W1^T), H2 = relu(H1 W2^T), Y = H2 W3^T
//                          (TextureMlp::forward, mlp.cpp:24-43)
//                 SH       dY = dL/dcoeffs from dL/drgb = w dL/dfinal + dL/dtexture
//                          (renderer.cpp:266-276; eval_sh_backward sh.hpp:76-83)
//                 backward dH2 = (dY W3) * [H2 > 0], dH1 = (dH2 W2) * [H1 > 0],
//                          dF = dH1 W1 (TextureMlp::backward, mlp.cpp:45-90)
//                 weights  gW3^T += H2^T dY, gW2 += dH2^T H1, gW1 += dH1^T F, K = the
//                          128 rows of the tile, accumulated in TMEM across all the
//                          tiles of the CTA; partials reduced in a fixed order at the end
//   S  scatter    one thread per slot: grid_lookup_backward (hash_grid.hpp:85-124):
//                 table gradients (exact order-independent accumulators, nx_xacc.cuh;
//                 warp-aggregated where the warp shares a cell), dL/dx, dL/dt ->
//                 d_t_slot = dL/dt + dot(dL/dx, dir)
//
// MMA operands are bf16 with the 3-term split (a.b ~ ah.bh + ah.bl + al.bh), as in
// the forward. The activations live in three combined K-major buffers so that every
// product — the row-wise chain (K = features) and the weight gradients (K = rows,
// operands read MN-major from the same bytes) — is one descriptor away:
//   C1 = [H2 | dH2]  (128 x 128)   C2 = [dY | H1]  (128 x 112)   C3 = [dH1 | F | pad]  (128 x 128)
//   G1 (TMEM cols 64..175)  = C1^T . C2 : rows 0..63 x cols 0..47 = gW3^T, rows 64..127 x cols 48..111 = gW2
//   G2 (TMEM cols 176..207) = C3^T . F  : rows 0..63 = gW1
// The backward chain reads the weight buffers MN-major too (B = W^T without a copy).
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "nx_composite.cuh"
#include "nx_grid.cuh"
#include "nx_tc.cuh"

namespace nx {

namespace {

constexpr int kThreadsM = 128;
constexpr int kRows = 128;
constexpr int kIn = 32, kHid = 64, kOut = 48;
constexpr int kC1 = 128, kC2 = 112, kC3 = 128;  // columns of the combined buffers
constexpr int kWGrads = kHid * kIn + kHid * kHid + kOut * kHid;  // 9216 partial values per CTA
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColD = 0, kColG1 = 64, kColG2 = 176;
// Per-slot scratch row (floats): [0, 32) features F, overwritten by dL/dF; [32, 37) the
// ReLU / SH-clamp masks of the exact fp32 forward (m1 lo/hi, m2 lo/hi, clamp bits).
constexpr int kStride = 40;

// shared-memory carve-up (bytes); every region 1 KB aligned
constexpr int kOffW1h = 0;
constexpr int kOffW1l = kOffW1h + kHid * kIn * 2;
constexpr int kOffW2h = kOffW1l + kHid * kIn * 2;
constexpr int kOffW2l = kOffW2h + kHid * kHid * 2;
constexpr int kOffW3h = kOffW2l + kHid * kHid * 2;
constexpr int kOffW3l = kOffW3h + kOut * kHid * 2;
constexpr int kOffC1h = kOffW3l + kOut * kHid * 2;
constexpr int kOffC1l = kOffC1h + kRows * kC1 * 2;
constexpr int kOffC2h = kOffC1l + kRows * kC1 * 2;
constexpr int kOffC2l = kOffC2h + kRows * kC2 * 2;
constexpr int kOffC3h = kOffC2l + kRows * kC2 * 2;
constexpr int kOffC3l = kOffC3h + kRows * kC3 * 2;
constexpr int kOffBar = kOffC3l + kRows * kC3 * 2;
constexpr int kOffTmem = kOffBar + 8;
constexpr int kSmemM = kOffTmem + 8;
static_assert(kSmemM <= 227 * 1024, "fits one CTA per SM");

// ---------------------------------------------------------------- G: features
// Per slot: the 16-level features F (grid_lookup) and, from the same gathered corners,
// the per-level sums the scatter's position / fade gradient needs (level_sums: the
// un-faded features and the trilinear Jacobian, 8 floats per level, level-major SoA
// jbuf[(l * 8 + k) * total + slot]), so that the table is gathered once per backward.
// The masks come next, from mask_tc_kernel.
__global__ void __launch_bounds__(128) features_kernel(const FieldBwdArgs a, const TcConst cst, float* __restrict__ fbuf,
                                                       float* __restrict__ jbuf, int64_t total) {
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (sl >= total) return;
    float feats[kIn];
#pragma unroll
    for (int i = 0; i < kIn; ++i) feats[i] = 0.f;
    if (a.fb.ids[sl] >= 0) {
        const int K = a.fb.K;
        const int64_t pix = sl / K;
        const int px = static_cast<int>(pix % a.cam.W), py = static_cast<int>(pix / a.cam.W);
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
                float js[8];
                level_sums(cur, js);
#pragma unroll
                for (int k = 0; k < 8; ++k) jbuf[static_cast<int64_t>(l * 8 + k) * total + sl] = js[k];
                if (l + 1 < kLevels) cur = nxt;
            }
        } else {
#pragma unroll
            for (int l = 0; l < kLevels; ++l) {
                const LevelFetch f = fetch_level<false>(l, x0, x1, x2, cst, tab, T, mask, ft, a.st.no_downweight);
                const float2 g = interp(f);
                feats[2 * l] = g.x;
                feats[2 * l + 1] = g.y;
                float js[8];
                level_sums(f, js);
#pragma unroll
                for (int k = 0; k < 8; ++k) jbuf[static_cast<int64_t>(l * 8 + k) * total + sl] = js[k];
            }
        }
    }
    float4* dst = reinterpret_cast<float4*>(fbuf + sl * kStride);
#pragma unroll
    for (int q = 0; q < kIn / 4; ++q) dst[q] = make_float4(feats[4 * q], feats[4 * q + 1], feats[4 * q + 2], feats[4 * q + 3]);
}

// The listed slots' masks re-decided with the reference's fp64 forward: grid_lookup
// (hash_grid.cpp:26-83) and TextureMlp::forward (mlp.cpp:24-43) in fp64, eval_sh_cached's
// clamp (sh.hpp:61-73). One warp per listed slot: lanes 0..15 take a level of the grid
// lookup each, then lane j forms outputs j and j + 32 of each layer — every dot product
// in the reference's order (inputs ascending), from transposed weights in shared memory
// (conflict-free) — and lane 0 sums the SH clamp terms in the reference's order.
constexpr int kMaskWarps = 4;
struct MaskSmem {
    float w1t[kIn][kHid];   // w1 transposed: [input][output]
    float w2t[kHid][kHid];
    float w3t[kHid][kOut];
    double x[kMaskWarps][kIn];
    double h1[kMaskWarps][kHid];
    double h2[kMaskWarps][kHid];
    double y[kMaskWarps][kOut];
};

__global__ void __launch_bounds__(32 * kMaskWarps) mask_fp64_kernel(const FieldBwdArgs a,
                                                                    const int32_t* __restrict__ amb_list,
                                                                    const int32_t* __restrict__ amb_count,
                                                                    float* __restrict__ fbuf) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    MaskSmem& sm = *reinterpret_cast<MaskSmem*>(smem_raw);
    for (int e = threadIdx.x; e < kHid * kIn; e += blockDim.x) sm.w1t[e % kIn][e / kIn] = __ldg(a.scene.w1 + e);
    for (int e = threadIdx.x; e < kHid * kHid; e += blockDim.x) sm.w2t[e % kHid][e / kHid] = __ldg(a.scene.w2 + e);
    for (int e = threadIdx.x; e < kOut * kHid; e += blockDim.x) sm.w3t[e % kHid][e / kHid] = __ldg(a.scene.w3 + e);
    __syncthreads();
    const int n = *amb_count;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const nx_field_desc& fd = a.scene.field;
    const uint32_t T = 1u << fd.log2_table, mask = T - 1u;
    double* x = sm.x[warp];
    double* h1 = sm.h1[warp];
    double* h2 = sm.h2[warp];
    double* y = sm.y[warp];
    for (int q = blockIdx.x * kMaskWarps + warp; q < n; q += gridDim.x * kMaskWarps) {
        const int64_t sl = amb_list[q];
        const int64_t pix = sl / a.fb.K;
        double dir[3];
        pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
        const double t = a.fb.depths[sl];
        if (lane < kLevels) {  // grid_lookup, level `lane`
            const int l = lane;
            double s = fd.base_scale;
            for (int k = 0; k < l; ++k) s *= fd.growth;  // the reference's iterated level scale
            const double x0 = a.cam.o[0] + t * dir[0], x1 = a.cam.o[1] + t * dir[1], x2 = a.cam.o[2] + t * dir[2];
            const double p0 = s * x0, p1 = s * x1, p2 = s * x2;
            const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
            const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                            b2 = static_cast<long long>(fl2);
            const double fr[3] = {p0 - fl0, p1 - fl1, p2 - fl2};
            double dw = 1.0;
            if (!a.st.no_downweight) {
                const double r = a.cam.fx / (s * t);
                dw = 1.0 - exp(-r * r / (2.0 * M_PI));
            }
            double g0 = 0.0, g1 = 0.0;
            for (int ci = 0; ci < 8; ++ci) {
                const uint32_t row = (map_positive32(b0 + (ci & 1)) ^ (map_positive32(b1 + ((ci >> 1) & 1)) * 2654435761u) ^
                                      (map_positive32(b2 + ((ci >> 2) & 1)) * 805459861u)) & mask;
                const double cw = ((ci & 1) ? fr[0] : 1.0 - fr[0]) * ((ci & 2) ? fr[1] : 1.0 - fr[1]) *
                                  ((ci & 4) ? fr[2] : 1.0 - fr[2]);
                const float2 v = __ldg(reinterpret_cast<const float2*>(a.scene.table) + static_cast<size_t>(l) * T + row);
                g0 += cw * v.x;
                g1 += cw * v.y;
            }
            x[2 * l] = g0 * dw;
            x[2 * l + 1] = g1 * dw;
        }
        __syncwarp();
        uint32_t m[4];
        {  // layer 1
            double a0 = 0.0, a1 = 0.0;
            for (int i = 0; i < kIn; ++i) {
                a0 += static_cast<double>(sm.w1t[i][lane]) * x[i];
                a1 += static_cast<double>(sm.w1t[i][lane + 32]) * x[i];
            }
            m[0] = __ballot_sync(0xffffffffu, a0 > 0.0);
            m[1] = __ballot_sync(0xffffffffu, a1 > 0.0);
            h1[lane] = a0 > 0.0 ? a0 : 0.0;
            h1[lane + 32] = a1 > 0.0 ? a1 : 0.0;
        }
        __syncwarp();
        {  // layer 2
            double a0 = 0.0, a1 = 0.0;
            for (int i = 0; i < kHid; ++i) {
                a0 += static_cast<double>(sm.w2t[i][lane]) * h1[i];
                a1 += static_cast<double>(sm.w2t[i][lane + 32]) * h1[i];
            }
            m[2] = __ballot_sync(0xffffffffu, a0 > 0.0);
            m[3] = __ballot_sync(0xffffffffu, a1 > 0.0);
            h2[lane] = a0 > 0.0 ? a0 : 0.0;
            h2[lane + 32] = a1 > 0.0 ? a1 : 0.0;
        }
        __syncwarp();
        {  // layer 3 (48 outputs)
            double a0 = 0.0, a1 = 0.0;
            for (int i = 0; i < kHid; ++i) {
                a0 += static_cast<double>(sm.w3t[i][lane]) * h2[i];
                if (lane < kOut - 32) a1 += static_cast<double>(sm.w3t[i][lane + 32]) * h2[i];
            }
            y[lane] = a0;
            if (lane < kOut - 32) y[lane + 32] = a1;
        }
        __syncwarp();
        if (lane == 0) {
            const double xx = dir[0] * dir[0], yy = dir[1] * dir[1], zz = dir[2] * dir[2];
            const double dx = dir[0], dy = dir[1], dz = dir[2];
            const double b[16] = {0.28209479177387814, -0.4886025119029199 * dy, 0.4886025119029199 * dz,
                                  -0.4886025119029199 * dx, 1.0925484305920792 * dx * dy, -1.0925484305920792 * dy * dz,
                                  0.31539156525252005 * (2.0 * zz - xx - yy), -1.0925484305920792 * dx * dz,
                                  0.5462742152960396 * (xx - yy), -0.5900435899266435 * dy * (3.0 * xx - yy),
                                  2.890611442640554 * dx * dy * dz, -0.4570457994644658 * dy * (4.0 * zz - xx - yy),
                                  0.3731763325901154 * dz * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                                  -0.4570457994644658 * dx * (4.0 * zz - xx - yy), 1.445305721320277 * dz * (xx - yy),
                                  -0.5900435899266435 * dx * (xx - 3.0 * yy)};
            double c3[3] = {0.5, 0.5, 0.5};
            for (int o = 0; o < kOut; ++o) c3[o % 3] += y[o] * b[o / 3];
            const uint32_t shm = (c3[0] >= 0.0 ? 1u : 0u) | (c3[1] >= 0.0 ? 2u : 0u) | (c3[2] >= 0.0 ? 4u : 0u);
            float4* dst = reinterpret_cast<float4*>(fbuf + sl * kStride);
            dst[kIn / 4] = make_float4(__uint_as_float(m[0]), __uint_as_float(m[1]), __uint_as_float(m[2]),
                                       __uint_as_float(m[3]));
            dst[kIn / 4 + 1] = make_float4(__uint_as_float(shm), 0.f, 0.f, 0.f);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- M: MLP forward + backward on tcgen05
// D = A . B^T over K, 3 split terms per 16-wide k-step. Descriptors: (start, lbo, sbo)
// and the byte advance per k-step of each operand.
struct Opnd {
    uint32_t hi, lo;   // smem addresses of the hi / lo copies (start of the sub-matrix)
    uint32_t lbo, sbo;
    uint32_t step;     // bytes to advance per 16-wide k-step
};

__device__ __forceinline__ void issue_mma(uint32_t dtm, const Opnd& A, const Opnd& B, int ksteps, uint32_t idesc,
                                          bool accumulate) {
    for (int s = 0; s < ksteps; ++s) {
        const uint32_t oa = s * A.step, ob = s * B.step;
        const uint64_t ah = smem_desc(A.hi + oa, A.lbo, A.sbo), al = smem_desc(A.lo + oa, A.lbo, A.sbo);
        const uint64_t bh = smem_desc(B.hi + ob, B.lbo, B.sbo), bl = smem_desc(B.lo + ob, B.lbo, B.sbo);
        mma_bf16(dtm, ah, bh, idesc, (accumulate || s > 0) ? 1u : 0u);
        mma_bf16(dtm, ah, bl, idesc, 1u);
        mma_bf16(dtm, al, bh, idesc, 1u);
    }
}

// K-major view of columns [c0, c0 + K) of a combined buffer with C columns (chain operand)
__device__ __forceinline__ Opnd kmaj(uint8_t* smem, int off_h, int off_l, int C, int c0) {
    const uint32_t base = (c0 / 8) * 128;
    return {smem_u32(smem + off_h) + base, smem_u32(smem + off_l) + base, 128u, static_cast<uint32_t>(16 * C), 256u};
}
// MN-major view (transposed operand) of columns [c0, ...) of a buffer with C columns:
// MN = columns (next 8 at 128 B), K = rows (next 8 at 16 C B)
__device__ __forceinline__ Opnd mnmaj(uint8_t* smem, int off_h, int off_l, int C, int c0) {
    const uint32_t base = (c0 / 8) * 128;
    return {smem_u32(smem + off_h) + base, smem_u32(smem + off_l) + base, static_cast<uint32_t>(16 * C), 128u,
            static_cast<uint32_t>(32 * C)};
}

__device__ __forceinline__ void load_weights_split(uint8_t* smem, const float* __restrict__ w, int rows, int K,
                                                   int off_h, int off_l) {
    for (int e = threadIdx.x; e < rows * K / 8; e += blockDim.x) {
        const int n = e / (K / 8), c = e % (K / 8);
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __ldg(w + n * K + c * 8 + i);
        store_split8(smem, off_h, off_l, kmajor_off(n, c * 8, K), x);
    }
}

__global__ void __launch_bounds__(kThreadsM, 1) mlp_bwd_tc_kernel(const FieldBwdArgs a, float* __restrict__ fbuf,
                                                                  float* __restrict__ partials, int64_t total,
                                                                  int64_t n_tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kOffBar);
    load_weights_split(smem, a.scene.w1, kHid, kIn, kOffW1h, kOffW1l);
    load_weights_split(smem, a.scene.w2, kHid, kHid, kOffW2h, kOffW2l);
    load_weights_split(smem, a.scene.w3, kOut, kHid, kOffW3h, kOffW3l);
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
    const uint32_t lane_off = static_cast<uint32_t>(32 * warp) << 16;
    const uint32_t tD = tmem + kColD + lane_off;
    uint32_t phase = 0;
    const int K = a.fb.K;
    const int row = tid;

    // operand views
    const Opnd W1k = kmaj(smem, kOffW1h, kOffW1l, kIn, 0), W2k = kmaj(smem, kOffW2h, kOffW2l, kHid, 0);
    const Opnd W1t = mnmaj(smem, kOffW1h, kOffW1l, kIn, 0), W2t = mnmaj(smem, kOffW2h, kOffW2l, kHid, 0),
               W3t = mnmaj(smem, kOffW3h, kOffW3l, kHid, 0);
    const Opnd F_k = kmaj(smem, kOffC3h, kOffC3l, kC3, 64), H1_k = kmaj(smem, kOffC2h, kOffC2l, kC2, 48),
               H2_k = kmaj(smem, kOffC1h, kOffC1l, kC1, 0), dY_k = kmaj(smem, kOffC2h, kOffC2l, kC2, 0),
               dH2_k = kmaj(smem, kOffC1h, kOffC1l, kC1, 64), dH1_k = kmaj(smem, kOffC3h, kOffC3l, kC3, 0);
    const Opnd C1_t = mnmaj(smem, kOffC1h, kOffC1l, kC1, 0), C2_t = mnmaj(smem, kOffC2h, kOffC2l, kC2, 0),
               C3_t = mnmaj(smem, kOffC3h, kOffC3l, kC3, 0), F_t = mnmaj(smem, kOffC3h, kOffC3l, kC3, 64);
    constexpr uint32_t kI64 = idesc_bf16_f32(kRows, 64);
    constexpr uint32_t kI64b = idesc_bf16_f32(kRows, 64, false, true), kI32b = idesc_bf16_f32(kRows, 32, false, true);
    constexpr uint32_t kIG1 = idesc_bf16_f32(kRows, kC2, true, true), kIG2 = idesc_bf16_f32(kRows, 32, true, true);

    bool first = true;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t sl = tile * kRows + row;
        const bool valid = sl < total && a.fb.ids[sl] >= 0;
        // ---- inputs of the row: features, dL/drgb, SH basis of the ray
        float x[kIn];
        float drgb[3] = {0.f, 0.f, 0.f};
        float b[16];
#pragma unroll
        for (int i = 0; i < kIn; ++i) x[i] = 0.f;
        uint64_t m1 = 0, m2 = 0;
        uint32_t shm = 0;
        if (valid) {
            const float4* src = reinterpret_cast<const float4*>(fbuf + sl * kStride);
#pragma unroll
            for (int q = 0; q < kIn / 4; ++q) {
                const float4 v = src[q];
                x[4 * q] = v.x;
                x[4 * q + 1] = v.y;
                x[4 * q + 2] = v.z;
                x[4 * q + 3] = v.w;
            }
            const float4 mk = src[kIn / 4];
            m1 = static_cast<uint64_t>(__float_as_uint(mk.x)) | (static_cast<uint64_t>(__float_as_uint(mk.y)) << 32);
            m2 = static_cast<uint64_t>(__float_as_uint(mk.z)) | (static_cast<uint64_t>(__float_as_uint(mk.w)) << 32);
            shm = __float_as_uint(src[kIn / 4 + 1].x);
            const int64_t pix = sl / K;
            const double w = a.fb.weights[sl];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double g = 0.0;
                if (a.d_final) g += w * a.d_final[pix * 3 + c];
                if (a.d_texture) g += a.d_texture[sl * 3 + c];
                drgb[c] = static_cast<float>(g);
            }
            double dir[3];
            pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
            const float dx = static_cast<float>(dir[0]), dy = static_cast<float>(dir[1]), dz = static_cast<float>(dir[2]);
            const float xx = dx * dx, yy = dy * dy, zz = dz * dz;
            b[0] = 0.28209479177387814f;
            b[1] = -0.4886025119029199f * dy;
            b[2] = 0.4886025119029199f * dz;
            b[3] = -0.4886025119029199f * dx;
            b[4] = 1.0925484305920792f * dx * dy;
            b[5] = -1.0925484305920792f * dy * dz;
            b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
            b[7] = -1.0925484305920792f * dx * dz;
            b[8] = 0.5462742152960396f * (xx - yy);
            b[9] = -0.5900435899266435f * dy * (3.0f * xx - yy);
            b[10] = 2.890611442640554f * dx * dy * dz;
            b[11] = -0.4570457994644658f * dy * (4.0f * zz - xx - yy);
            b[12] = 0.3731763325901154f * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = -0.4570457994644658f * dx * (4.0f * zz - xx - yy);
            b[14] = 1.445305721320277f * dz * (xx - yy);
            b[15] = -0.5900435899266435f * dx * (xx - 3.0f * yy);
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) b[k] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < kIn / 8; ++c) store_split8(smem, kOffC3h, kOffC3l, kmajor_off(row, 64 + 8 * c, kC3), x + 8 * c);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();

        // ---- L1: D = F . W1^T -> H1 = relu -> C2[:, 48..111]
        if (tid == 0) {
            tc_fence_after();
            issue_mma(tmem + kColD, F_k, W1k, kIn / 16, kI64, false);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kHid / 16; ++c) {
            float v[16];
            tmem_ld16(tD + 16 * c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
            store_split8(smem, kOffC2h, kOffC2l, kmajor_off(row, 48 + 16 * c, kC2), v);
            store_split8(smem, kOffC2h, kOffC2l, kmajor_off(row, 48 + 16 * c + 8, kC2), v + 8);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        // ---- L2: D = H1 . W2^T -> H2 -> C1[:, 0..63]
        if (tid == 0) {
            tc_fence_after();
            issue_mma(tmem + kColD, H1_k, W2k, kHid / 16, kI64, false);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kHid / 16; ++c) {
            float v[16];
            tmem_ld16(tD + 16 * c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
            store_split8(smem, kOffC1h, kOffC1l, kmajor_off(row, 16 * c, kC1), v);
            store_split8(smem, kOffC1h, kOffC1l, kmajor_off(row, 16 * c + 8, kC1), v + 8);
        }
        // ---- dY = dL/dcoeffs (eval_sh_backward, sh.hpp:76-83) with the exact clamp mask -> C2[:, 0..47]
        // (the coefficients themselves are not needed: Y only decides the clamp mask)
        {
            float dyv[kOut];
#pragma unroll
            for (int o = 0; o < kOut; ++o) dyv[o] = (shm >> (o % 3)) & 1u ? drgb[o % 3] * b[o / 3] : 0.f;
#pragma unroll
            for (int c = 0; c < kOut / 8; ++c) store_split8(smem, kOffC2h, kOffC2l, kmajor_off(row, 8 * c, kC2), dyv + 8 * c);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        // ---- dH2 = (dY . W3) * [H2 > 0] -> C1[:, 64..127]
        if (tid == 0) {
            tc_fence_after();
            issue_mma(tmem + kColD, dY_k, W3t, kOut / 16, kI64b, false);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kHid / 16; ++c) {
            float v[16];
            tmem_ld16(tD + 16 * c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = (m2 >> (16 * c + i)) & 1ull ? v[i] : 0.f;
            store_split8(smem, kOffC1h, kOffC1l, kmajor_off(row, 64 + 16 * c, kC1), v);
            store_split8(smem, kOffC1h, kOffC1l, kmajor_off(row, 64 + 16 * c + 8, kC1), v + 8);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        // ---- G1 += C1^T . C2 (gW3^T, gW2); dH1 = (dH2 . W2) * [H1 > 0] -> C3[:, 0..63]
        if (tid == 0) {
            tc_fence_after();
            issue_mma(tmem + kColG1, C1_t, C2_t, kRows / 16, kIG1, !first);
            issue_mma(tmem + kColD, dH2_k, W2t, kHid / 16, kI64b, false);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < kHid / 16; ++c) {
            float v[16];
            tmem_ld16(tD + 16 * c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = (m1 >> (16 * c + i)) & 1ull ? v[i] : 0.f;
            store_split8(smem, kOffC3h, kOffC3l, kmajor_off(row, 16 * c, kC3), v);
            store_split8(smem, kOffC3h, kOffC3l, kmajor_off(row, 16 * c + 8, kC3), v + 8);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        // ---- G2 += C3^T . F (gW1); dF = dH1 . W1
        if (tid == 0) {
            tc_fence_after();
            issue_mma(tmem + kColG2, C3_t, F_t, kRows / 16, kIG2, !first);
            issue_mma(tmem + kColD, dH1_k, W1t, kHid / 16, kI32b, false);
            mma_commit(bar);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
        {
            float v[kIn];
            tmem_ld16(tD, v);
            tmem_ld16(tD + 16, v + 16);
            if (valid) {
                float4* dst = reinterpret_cast<float4*>(fbuf + sl * kStride);
#pragma unroll
                for (int q = 0; q < kIn / 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
        }
        tc_fence_before();
        __syncthreads();  // the next tile rewrites C1..C3 only after every MMA above completed
        first = false;
    }
    // ---- weight-gradient partials of this CTA: [w1 (64x32) | w2 (64x64) | w3 (48x64)]
    tc_fence_after();
    float* part = partials + static_cast<int64_t>(blockIdx.x) * kWGrads;
    float* p1 = part;
    float* p2 = part + kHid * kIn;
    float* p3 = p2 + kHid * kHid;
    float g1[kC2], g2[32];
#pragma unroll
    for (int c = 0; c < kC2 / 16; ++c) tmem_ld16(tmem + kColG1 + lane_off + 16 * c, g1 + 16 * c);
    tmem_ld16(tmem + kColG2 + lane_off, g2);
    tmem_ld16(tmem + kColG2 + lane_off + 16, g2 + 16);
    if (first) {  // no tile: the accumulators were never written
#pragma unroll
        for (int i = 0; i < kC2; ++i) g1[i] = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) g2[i] = 0.f;
    }
    if (row < kHid) {
#pragma unroll
        for (int o = 0; o < kOut; ++o) p3[o * kHid + row] = g1[o];  // gW3[o][i = row]
#pragma unroll
        for (int i = 0; i < kIn; ++i) p1[row * kIn + i] = g2[i];    // gW1[o = row][i]
    } else {
#pragma unroll
        for (int i = 0; i < kHid; ++i) p2[(row - kHid) * kHid + i] = g1[48 + i];  // gW2[o = row-64][i]
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------- M0: ReLU / clamp masks on tcgen05
// The masks (which ReLU units and SH-clamped channels pass gradients, mlp.cpp:67-68,
// 79-80; sh.hpp:70) from a tensor-core forward of the features F at fp32 accuracy:
// every operand is split three ways (x = h + m + l in bf16, 24 significant bits) and
// each product is formed from the six terms above 2^-24 (hh, hm, mh, hl, lh, mm), so
// the pre-activations carry the error of an fp32 forward. As before (an fp32 CUDA-core
// forward, profiles/r01), a unit whose pre-activation lies within 2^-15 ||a||_1 max|w_o|
// of the threshold (SH: 2^-14 ||h2||_1 max|w3| sum|b|) is "ambiguous": the slot is
// listed and mask_fp64_kernel re-decides it with the reference's fp64 forward.
struct Opnd3 {
    uint32_t p[3];  // hi, mid, lo copies
    uint32_t lbo, sbo, step;
};
constexpr int kM3W1 = 0;                                // 3 x [64][32]
constexpr int kM3W2 = kM3W1 + 3 * kHid * kIn * 2;       // 3 x [64][64]
constexpr int kM3W3 = kM3W2 + 3 * kHid * kHid * 2;      // 3 x [48][64]
constexpr int kM3A = kM3W3 + 3 * kOut * kHid * 2;       // 3 x [128][64] (F in columns 0..31)
constexpr int kM3Max = kM3A + 3 * kRows * kHid * 2;     // per-row weight maxima
constexpr int kM3Bar = kM3Max + 1024;
constexpr int kM3Tmem = kM3Bar + 8;
constexpr int kSmemMask = kM3Tmem + 8;
constexpr uint32_t kMaskTmemCols = 64;
static_assert(kSmemMask <= 113 * 1024, "two CTAs per SM");

// 8 consecutive K values as three bf16 parts (exact re-expansion of each part by shifts)
__device__ __forceinline__ void store_split3x8(uint8_t* smem, int off, int part_bytes, uint32_t byte_off,
                                               const float* x) {
    uint32_t h[4], m[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = pack_bf16(x[2 * i], x[2 * i + 1]);
        const float r0 = x[2 * i] - __uint_as_float(h[i] << 16), r1 = x[2 * i + 1] - __uint_as_float(h[i] & 0xffff0000u);
        m[i] = pack_bf16(r0, r1);
        l[i] = pack_bf16(r0 - __uint_as_float(m[i] << 16), r1 - __uint_as_float(m[i] & 0xffff0000u));
    }
    *reinterpret_cast<uint4*>(smem + off + byte_off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(smem + off + part_bytes + byte_off) = make_uint4(m[0], m[1], m[2], m[3]);
    *reinterpret_cast<uint4*>(smem + off + 2 * part_bytes + byte_off) = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ Opnd3 kmaj3(uint8_t* smem, int off, int part_bytes, int C) {
    const uint32_t b = smem_u32(smem + off);
    return {{b, b + static_cast<uint32_t>(part_bytes), b + 2u * static_cast<uint32_t>(part_bytes)},
            128u, static_cast<uint32_t>(16 * C), 256u};
}

__device__ __forceinline__ void issue_mma3(uint32_t dtm, const Opnd3& A, const Opnd3& B, int ksteps, uint32_t idesc) {
    constexpr int kTerms[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};
    for (int s = 0; s < ksteps; ++s) {
#pragma unroll
        for (int t = 0; t < 6; ++t) {
            const uint64_t da = smem_desc(A.p[kTerms[t][0]] + s * A.step, A.lbo, A.sbo);
            const uint64_t db = smem_desc(B.p[kTerms[t][1]] + s * B.step, B.lbo, B.sbo);
            mma_bf16(dtm, da, db, idesc, (s > 0 || t > 0) ? 1u : 0u);
        }
    }
}

__global__ void __launch_bounds__(kThreadsM) mask_tc_kernel(const FieldBwdArgs a, float* __restrict__ fbuf,
                                                            int64_t total, int64_t n_tiles,
                                                            int32_t* __restrict__ amb_list,
                                                            int32_t* __restrict__ amb_count) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bar = smem_u32(smem + kM3Bar);
    const float* wsrc[3] = {a.scene.w1, a.scene.w2, a.scene.w3};
    const int wrows[3] = {kHid, kHid, kOut}, wk[3] = {kIn, kHid, kHid}, woff[3] = {kM3W1, kM3W2, kM3W3};
#pragma unroll 1
    for (int m = 0; m < 3; ++m)
        for (int e = tid; e < wrows[m] * wk[m] / 8; e += blockDim.x) {
            const int n = e / (wk[m] / 8), c = e % (wk[m] / 8);
            float x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __ldg(wsrc[m] + n * wk[m] + c * 8 + i);
            store_split3x8(smem, woff[m], wrows[m] * wk[m] * 2, kmajor_off(n, c * 8, wk[m]), x);
        }
    float* sMax = reinterpret_cast<float*>(smem + kM3Max);  // [0,64) w1 rows, [64,128) w2 rows, 128: w3
    for (int o = tid; o < 2 * kHid + 1; o += blockDim.x) {
        float mx = 0.f;
        if (o < kHid)
            for (int i = 0; i < kIn; ++i) mx = fmaxf(mx, fabsf(__ldg(a.scene.w1 + o * kIn + i)));
        else if (o < 2 * kHid)
            for (int i = 0; i < kHid; ++i) mx = fmaxf(mx, fabsf(__ldg(a.scene.w2 + (o - kHid) * kHid + i)));
        else
            for (int i = 0; i < kOut * kHid; ++i) mx = fmaxf(mx, fabsf(__ldg(a.scene.w3 + i)));
        sMax[o] = mx;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem + kM3Tmem)),
                     "r"(kMaskTmemCols));
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
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + kM3Tmem);
    const uint32_t tD = tmem + (static_cast<uint32_t>(32 * warp) << 16);
    constexpr int kAPart = kRows * kHid * 2;
    const Opnd3 A = kmaj3(smem, kM3A, kAPart, kHid);
    const Opnd3 W1k = kmaj3(smem, kM3W1, kHid * kIn * 2, kIn), W2k = kmaj3(smem, kM3W2, kHid * kHid * 2, kHid),
                W3k = kmaj3(smem, kM3W3, kOut * kHid * 2, kHid);
    constexpr uint32_t kI64 = idesc_bf16_f32(kRows, 64), kI48 = idesc_bf16_f32(kRows, 48);
    const float max3 = sMax[2 * kHid];
    uint32_t phase = 0;
    const int row = tid;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t sl = tile * kRows + row;
        const bool valid = sl < total && a.fb.ids[sl] >= 0;
        float x[kIn];
        float n1 = 0.f;
        if (valid) {
            const float4* src = reinterpret_cast<const float4*>(fbuf + sl * kStride);
#pragma unroll
            for (int q = 0; q < kIn / 4; ++q) {
                const float4 v = src[q];
                x[4 * q] = v.x;
                x[4 * q + 1] = v.y;
                x[4 * q + 2] = v.z;
                x[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kIn; ++i) x[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < kIn; ++i) n1 += fabsf(x[i]);
#pragma unroll
        for (int c = 0; c < kIn / 8; ++c) store_split3x8(smem, kM3A, kAPart, kmajor_off(row, 8 * c, kHid), x + 8 * c);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            issue_mma3(tmem, A, W1k, kIn / 16, kI64);
            mma_commit(bar);
        }
        // the ray's SH basis while layer 1 runs
        float b[16];
        {
            double dir[3] = {0.0, 0.0, 1.0};
            if (valid) {
                const int64_t pix = sl / a.fb.K;
                pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
            }
            sh_basis_f32(static_cast<float>(dir[0]), static_cast<float>(dir[1]), static_cast<float>(dir[2]), b);
        }
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
        uint32_t m1[2] = {0u, 0u}, m2[2] = {0u, 0u};
        bool amb = false;
        float nin = n1;
#pragma unroll
        for (int layer = 0; layer < 2; ++layer) {
            const float* rmax = sMax + layer * kHid;
            const float scale = 3.05e-5f * nin;
            float nout = 0.f;
#pragma unroll
            for (int c = 0; c < kHid / 16; ++c) {
                float v[16];
                tmem_ld16(tD + 16 * c, v);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int o = 16 * c + i;
                    if (v[i] > 0.f) (layer == 0 ? m1 : m2)[o >> 5] |= 1u << (o & 31);
                    amb |= fabsf(v[i]) <= scale * rmax[o];
                    v[i] = fmaxf(v[i], 0.f);
                    nout += v[i];
                }
                store_split3x8(smem, kM3A, kAPart, kmajor_off(row, 16 * c, kHid), v);
                store_split3x8(smem, kM3A, kAPart, kmajor_off(row, 16 * c + 8, kHid), v + 8);
            }
            nin = nout;
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                tc_fence_after();
                if (layer == 0) issue_mma3(tmem, A, W2k, kHid / 16, kI64);
                else issue_mma3(tmem, A, W3k, kHid / 16, kI48);
                mma_commit(bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        // eval_sh_cached's clamp (sh.hpp:61-73): 0.5 + sum_k Y[3k + c] b_k >= 0
        float c3[3] = {0.5f, 0.5f, 0.5f}, bsum = 0.f;
#pragma unroll
        for (int c = 0; c < kOut / 16; ++c) {
            float v[16];
            tmem_ld16(tD + 16 * c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int o = 16 * c + i;
                c3[o % 3] = fmaf(v[i], b[o / 3], c3[o % 3]);
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) bsum += fabsf(b[k]);
        const float bound3 = 6.1e-5f * nin * max3 * bsum;
        const uint32_t shm = (c3[0] >= 0.f ? 1u : 0u) | (c3[1] >= 0.f ? 2u : 0u) | (c3[2] >= 0.f ? 4u : 0u);
        amb |= fabsf(c3[0]) <= bound3 || fabsf(c3[1]) <= bound3 || fabsf(c3[2]) <= bound3;
        if (valid) {
            float4* dst = reinterpret_cast<float4*>(fbuf + sl * kStride);
            dst[kIn / 4] = make_float4(__uint_as_float(m1[0]), __uint_as_float(m1[1]), __uint_as_float(m2[0]),
                                       __uint_as_float(m2[1]));
            dst[kIn / 4 + 1] = make_float4(__uint_as_float(shm), 0.f, 0.f, 0.f);
            if (amb) amb_list[atomicAdd(amb_count, 1)] = static_cast<int32_t>(sl);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kMaskTmemCols));
}

// Sums the CTA partials in CTA order (deterministic) into the fp64 weight gradients.
__global__ void reduce_wgrads_kernel(const float* __restrict__ partials, int n_parts, double* g_w1, double* g_w2,
                                     double* g_w3) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kWGrads) return;
    double s = 0.0;
    for (int p = 0; p < n_parts; ++p) s += partials[static_cast<int64_t>(p) * kWGrads + i];
    if (i < kHid * kIn) g_w1[i] += s;
    else if (i < kHid * kIn + kHid * kHid) g_w2[i - kHid * kIn] += s;
    else g_w3[i - kHid * kIn - kHid * kHid] += s;
}

// ---------------------------------------------------------------- S: grid_lookup_backward
// grid_lookup_backward (hash_grid.hpp:85-124) in two phases: (1) the position / fade
// gradient from the per-level sums the features pass kept (jbuf: no second table
// gather); (2) the table gradients, which need only the corner rows and weights — into
// exact accumulators (nx_xacc.cuh), so that the table gradients do not
// depend on the order of the atomics. Neighbouring slots of a warp share corner rows at
// every level but the very finest (a warp covers 16 adjacent pixels), so the lanes that
// hit the same row (__match_any_sync) are summed first, in lane order, and their leader
// adds the sum: one accumulator update per distinct row of the warp.
__device__ __forceinline__ void scatter_dt(const FieldBwdArgs& a, const TcConst& cst, bool valid, float ft,
                                           const float* g, double t, double* dx, double& dt,
                                           const float* __restrict__ jbuf, int64_t total, int64_t slot) {
    // ---- phase 1: d_x, d_t from the kept sums: dL/dp_d = dw (g . J_d), dL/d(dw) = g . S
    // fade t-gradient (hash_grid.hpp:117-121): r^2 / (pi t) with r = fx / (s t) is
    // fx^2 / (pi t^3) / s^2 — one division per slot (a gradient value, no decision)
    const double fade_c = a.cam.fx * a.cam.fx / (M_PI * t * t * t);
    if (valid) {
#pragma unroll 4
        for (int l = 0; l < kLevels; ++l) {
            float js[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) js[k] = __ldg(jbuf + static_cast<int64_t>(l * 8 + k) * total + slot);
            const float g0 = g[2 * l], g1 = g[2 * l + 1];
            const float dw = level_fade(l, cst, ft, a.st.no_downweight);
            const float dp0 = dw * (g0 * js[2] + g1 * js[5]), dp1 = dw * (g0 * js[3] + g1 * js[6]),
                        dp2 = dw * (g0 * js[4] + g1 * js[7]);
            const float d_dw = g0 * js[0] + g1 * js[1];
            const double sl = cst.level_scale[l];
            dx[0] += sl * dp0;
            dx[1] += sl * dp1;
            dx[2] += sl * dp2;
            if (!a.st.no_downweight) {
                // downweight_grad_t via the cached factor (hash_grid.hpp:117-121)
                dt += static_cast<double>(d_dw) * (static_cast<double>(dw) - 1.0) * fade_c * cst.inv_level_scale2[l];
            }
        }
    }
}

template <bool kSmall>
__device__ __forceinline__ void scatter_table(const FieldBwdArgs& a, const TcConst& cst, bool valid, double x0,
                                              double x1, double x2, float ft, const float* g, const Xacc& tacc,
                                              float2* __restrict__ wsh) {
    const uint32_t T = 1u << a.scene.field.log2_table, mask = T - 1u;
    const int lane = threadIdx.x & 31;
    // ---- phase 2: table gradients dL/dtable[row][f] += g[f] * dw * corner_w (hash_grid.hpp:99-103)
#pragma unroll 1
    for (int l = 0; l < kLevels; ++l) {
        const LevelCell c = level_cell<kSmall>(l, x0, x1, x2, cst, mask, ft, a.st.no_downweight);
        const float g0 = valid ? g[2 * l] * c.dw : 0.f, g1 = valid ? g[2 * l + 1] * c.dw : 0.f;
        const float wx[2] = {1.0f - c.fr0, c.fr0}, wy[2] = {1.0f - c.fr1, c.fr1}, wz[2] = {1.0f - c.fr2, c.fr2};
        const int64_t slab = static_cast<int64_t>(l) * T * 2;
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
            const float cw = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
            const float u0 = g0 * cw, u1 = g1 * cw;
            const uint32_t key = valid ? c.row[ci] : 0xffffffffu;
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const uint32_t leaders = __ballot_sync(0xffffffffu, valid && lane == __ffs(peers) - 1);
            const int max_size = __reduce_max_sync(0xffffffffu, valid ? __popc(peers) : 0);
            float my0 = 0.f, my1 = 0.f;  // this lane's group sum when it leads a group
            if (__popc(leaders) * 4 <= max_size) {
                // few large groups (coarse levels): one warp-wide tree sum per group
                for (uint32_t L = leaders; L; L &= L - 1) {
                    const int ld = __ffs(L) - 1;
                    const bool mine = key == __shfl_sync(0xffffffffu, key, ld);
                    float s0 = mine ? u0 : 0.f, s1 = mine ? u1 : 0.f;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                    }
                    if (lane == ld) {
                        my0 = s0;
                        my1 = s1;
                    }
                }
            } else {
                // many small groups (fine levels): each leader sums its group in lane order
                wsh[lane] = make_float2(u0, u1);
                __syncwarp();
                if (valid && lane == __ffs(peers) - 1)
                    for (uint32_t m = peers; m;) {
                        // four members per round: independent loads, adds still in lane order
                        int idx[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            idx[q] = __ffs(m) - 1;
                            m &= m - 1;
                        }
                        float2 u[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) u[q] = wsh[idx[q] < 0 ? 0 : idx[q]];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (idx[q] >= 0) {
                                my0 += u[q].x;
                                my1 += u[q].y;
                            }
                    }
                __syncwarp();
            }
            if (valid && lane == __ffs(peers) - 1) {  // one accumulator update per distinct row
                const int64_t dst = slab + static_cast<int64_t>(c.row[ci]) * 2;
                xacc_add(tacc, dst, my0);
                xacc_add(tacc, dst + 1, my1);
            }
        }
    }
}

// per slot: the query point, its ray and dL/dF (fbuf); false for an empty slot
__device__ __forceinline__ bool scatter_slot(const FieldBwdArgs& a, const float* __restrict__ fbuf, int64_t sl,
                                             int64_t total, double* dir, double& t, double* x, float* g) {
    dir[0] = 0.0;
    dir[1] = 0.0;
    dir[2] = 1.0;
    t = 1.0;
    x[0] = x[1] = x[2] = 0.0;
#pragma unroll
    for (int i = 0; i < kIn; ++i) g[i] = 0.f;
    if (sl >= total || a.fb.ids[sl] < 0) return false;
    const int64_t pix = sl / a.fb.K;
    pixel_dir(a.cam, static_cast<int>(pix % a.cam.W) + 0.5, static_cast<int>(pix / a.cam.W) + 0.5, dir);
    t = a.fb.depths[sl];
    x[0] = a.cam.o[0] + t * dir[0];
    x[1] = a.cam.o[1] + t * dir[1];
    x[2] = a.cam.o[2] + t * dir[2];
    const float4* src = reinterpret_cast<const float4*>(fbuf + sl * kStride);
#pragma unroll
    for (int q = 0; q < kIn / 4; ++q) {
        const float4 v = src[q];
        g[4 * q] = v.x;
        g[4 * q + 1] = v.y;
        g[4 * q + 2] = v.z;
        g[4 * q + 3] = v.w;
    }
    return true;
}

// S1: d_t_slot = dL/dt + dot(dL/dx, dir) (renderer.cpp:283-284) — what the compositing
// branch needs; the table gradients (S2) can then run beside it
__global__ void __launch_bounds__(128) scatter_dt_kernel(const FieldBwdArgs a, const TcConst cst,
                                                         const float* __restrict__ fbuf, int64_t total,
                                                         const float* __restrict__ jbuf) {
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double dir[3], t, x[3];
    float g[kIn];
    const bool valid = scatter_slot(a, fbuf, sl, total, dir, t, x, g);
    if (!valid) {
        if (sl < total) a.d_t_slot[sl] = 0.0;
        return;
    }
    const float ft = static_cast<float>(a.cam.fx / t);
    double dx[3] = {0.0, 0.0, 0.0}, dt = 0.0;
    scatter_dt(a, cst, true, ft, g, t, dx, dt, jbuf, total, sl);
    a.d_t_slot[sl] = dt + (dx[0] * dir[0] + dx[1] * dir[1] + dx[2] * dir[2]);
}

// S2: the table gradients
#ifndef NX_SCATTER_MINB
#define NX_SCATTER_MINB 1
#endif
__global__ void __launch_bounds__(128, NX_SCATTER_MINB) scatter_table_kernel(const FieldBwdArgs a, const TcConst cst,
                                                            const float* __restrict__ fbuf, int64_t total,
                                                            const Xacc tacc) {
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double dir[3], t, x[3];
    float g[kIn];
    const bool valid = scatter_slot(a, fbuf, sl, total, dir, t, x, g);
    if (!__any_sync(0xffffffffu, valid)) return;
    __shared__ float2 wsh[128];
    const float ft = static_cast<float>(a.cam.fx / t);
    const bool small = fmax(fabs(x[0]), fmax(fabs(x[1]), fabs(x[2]))) * cst.level_scale[kLevels - 1] < 1073741824.0;
    if (__all_sync(0xffffffffu, small))
        scatter_table<true>(a, cst, valid, x[0], x[1], x[2], ft, g, tacc, wsh + (threadIdx.x & ~31));
    else
        scatter_table<false>(a, cst, valid, x[0], x[1], x[2], ft, g, tacc, wsh + (threadIdx.x & ~31));
}

}  // namespace

// g_table += the exact table-gradient sums (and clears the accumulators for the next call).
__global__ void take_table_kernel(double* __restrict__ g, const Xacc acc) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < acc.m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = xacc_take(acc, i);
        if (v != 0.0) g[i] += v;
    }
}

namespace {


}  // namespace

bool field_backward_tc_supported(const nx_field_desc& fd) {
    return fd.levels == kLevels && fd.features == 2 && fd.n_hidden == kHid;
}

int launch_field_backward_tc(const FieldBwdArgs& a, cudaStream_t s) {
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * a.fb.K;
    if (total == 0) return NX_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    FieldBwdScratch& sc = *a.scratch;
    const size_t fneed = static_cast<size_t>(total) * kStride;
    const int64_t n_tiles = (total + kRows - 1) / kRows;
    const int grid_m = static_cast<int>(std::min<int64_t>(n_tiles, sms));
    const size_t pneed = static_cast<size_t>(grid_m) * kWGrads;
    if (fneed > sc.fcap) {
        if (sc.fbuf) cudaFree(sc.fbuf);
        sc.fbuf = nullptr;
        sc.fcap = 0;
        if (cudaMalloc(&sc.fbuf, fneed * sizeof(float)) != cudaSuccess) return NX_OUT_OF_MEMORY;
        sc.fcap = fneed;
    }
    if (static_cast<size_t>(total) + 1 > sc.acap) {
        if (sc.amb) cudaFree(sc.amb);
        sc.amb = nullptr;
        sc.acap = 0;
        if (cudaMalloc(&sc.amb, (total + 1) * sizeof(int32_t)) != cudaSuccess) return NX_OUT_OF_MEMORY;
        sc.acap = total + 1;
    }
    const int64_t tneed = static_cast<int64_t>(kLevels) * (int64_t(1) << a.scene.field.log2_table) * 2;
    if (int st = sc.table_acc(tneed, s)) return st;
    const size_t jneed = static_cast<size_t>(total) * kLevels * 8;
    if (jneed > sc.jcap) {
        if (sc.jbuf) cudaFree(sc.jbuf);
        sc.jbuf = nullptr;
        sc.jcap = 0;
        if (cudaMalloc(&sc.jbuf, jneed * sizeof(float)) != cudaSuccess) return NX_OUT_OF_MEMORY;
        sc.jcap = jneed;
    }
    if (pneed > sc.pcap) {
        if (sc.parts) cudaFree(sc.parts);
        sc.parts = nullptr;
        sc.pcap = 0;
        if (cudaMalloc(&sc.parts, pneed * sizeof(float)) != cudaSuccess) return NX_OUT_OF_MEMORY;
        sc.pcap = pneed;
    }
    TcConst cst;
    double scale = a.scene.field.base_scale;
    for (int l = 0; l < kLevels; ++l, scale *= a.scene.field.growth) {
        cst.level_scale[l] = scale;
        cst.inv_level_scale[l] = static_cast<float>(1.0 / scale);
        cst.inv_level_scale2[l] = 1.0 / (scale * scale);
    }
    const unsigned blocks = static_cast<unsigned>((total + 127) / 128);
    count_launch(6);
    cudaMemsetAsync(sc.amb, 0, sizeof(int32_t), s);
    features_kernel<<<blocks, 128, 0, s>>>(a, cst, sc.fbuf, sc.jbuf, total);
    cudaFuncSetAttribute(mask_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMask);
    mask_tc_kernel<<<static_cast<unsigned>(std::min<int64_t>(n_tiles, 2 * sms)), kThreadsM, kSmemMask, s>>>(
        a, sc.fbuf, total, n_tiles, sc.amb + 1, sc.amb);
    cudaFuncSetAttribute(mask_fp64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(MaskSmem)));
    mask_fp64_kernel<<<4 * sms, 32 * kMaskWarps, sizeof(MaskSmem), s>>>(a, sc.amb + 1, sc.amb, sc.fbuf);
    cudaFuncSetAttribute(mlp_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemM);
    mlp_bwd_tc_kernel<<<grid_m, kThreadsM, kSmemM, s>>>(a, sc.fbuf, sc.parts, total, n_tiles);
    reduce_wgrads_kernel<<<(kWGrads + 255) / 256, 256, 0, s>>>(sc.parts, grid_m, a.g_w1, a.g_w2, a.g_w3);
    const Xacc tacc{sc.tx, tneed};
    scatter_dt_kernel<<<blocks, 128, 0, s>>>(a, cst, sc.fbuf, total, sc.jbuf);
    // the table gradients beside the compositing branch (which needs d_t_slot only)
    cudaStream_t st = s;
    if (a.side && a.ev_fork && a.ev_join) {
        cudaEventRecord(a.ev_fork, s);
        cudaStreamWaitEvent(a.side, a.ev_fork, 0);
        st = a.side;
    }
    count_launch(2);
    scatter_table_kernel<<<blocks, 128, 0, st>>>(a, cst, sc.fbuf, total, tacc);
    take_table_kernel<<<8 * sms, 256, 0, st>>>(a.g_table, tacc);
    if (st != s) cudaEventRecord(a.ev_join, st);
    return NX_OK;
}

}  // namespace nx
