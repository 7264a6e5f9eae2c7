// K6 composite: per-tile front-to-back alpha compositing with early termination
// and a top-K buffer (collection_pass, renderer.cpp:115-171).
//
// One CTA per screen tile, one thread per pixel. The tile's work list (ids in
// (depth, id) order) is walked in chunks of kChunk primitives whose records are
// staged into shared memory. Per chunk, each pixel
//   A. runs an fp32 conservative prefilter over every primitive of the chunk
//      (broadcast smem reads, no divergence) and records the survivors in a
//      128-bit mask: a test is dropped only if it provably fails the reference's
//      t > near_eps or |u| <= ru, |v| <= rv conditions (hence alpha < 1/255),
//      with a rigorous fp32 error slack;
//   B. walks its own survivors in list order on the exact fp64 path — the
//      reference's intersect() formulas (intersect.hpp:23-42), eval_kernel, the
//      1/255 test, alpha clamp, top-K insert, transmittance update and
//      termination (renderer.cpp:144-153).
// Lanes walk their own survivor queues in lockstep, so a warp pays for the
// longest queue of its pixels instead of the union of all their hits. Every
// decision is taken in fp64 with the reference formulas; the prefilter only
// skips provable misses, so contributor lists are bit-exact.
#include "nx_fp64math.h"
#include "nx_internal.cuh"

namespace nx {

namespace {

constexpr int kThreads = 256;
constexpr int kChunk = 128;
constexpr int kRecPairs = REC_FIELDS / 2;      // double2 per fp64 record (10)
constexpr int kRecStride = kRecPairs + 1;      // padded to 11 double2 (176 B): lanes reading
                                               // different records hit different bank groups

// Primitive SH colour (eval_sh, sh.hpp:46-57) in fp32 from the ray direction:
// colour outputs are tolerance-checked (max-abs 1e-3), decisions never use it.
__device__ __forceinline__ void eval_sh_f32(const float* __restrict__ sh, float x, float y, float z, int degree,
                                            float* rgb) {
    float a0 = 0.5f + 0.28209479177387814f * __ldg(sh + 0);
    float a1 = 0.5f + 0.28209479177387814f * __ldg(sh + 1);
    float a2 = 0.5f + 0.28209479177387814f * __ldg(sh + 2);
    if (degree >= 3) {
        const float xx = x * x, yy = y * y, zz = z * z;
        float b[16];
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
    rgb[0] = fmaxf(a0, 0.f);
    rgb[1] = fmaxf(a1, 0.f);
    rgb[2] = fmaxf(a2, 0.f);
}

// fp32 conservative prefilter: false only if the exact test provably misses.
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

template <int K, bool kDebug>
__global__ void __launch_bounds__(kThreads, 2) composite_kernel(const CompositeArgs a) {
    constexpr int KK = K > 0 ? K : 1;
    __shared__ float4 s_f[kChunk][4];
    __shared__ double2 s_d[kChunk][kRecStride];
    __shared__ int32_t s_id[kChunk];

    const int tile = a.st.tile;
    const int t = blockIdx.x;
    const int tx = t % a.fb.tiles_x, ty = t / a.fb.tiles_x;
    const int list_begin = a.tile_offsets[t], list_end = a.tile_offsets[t + 1];
    const int W = a.cam.W, H = a.cam.H;
    const double near_eps = a.st.near_eps, alpha_max = a.st.alpha_max, min_T = a.st.min_transmittance;
    const float near_eps_f = static_cast<float>(near_eps);

    for (int pbase = 0; pbase < tile * tile; pbase += kThreads) {
        const int lp = pbase + threadIdx.x;
        const int px = tx * tile + lp % tile, py = ty * tile + lp / tile;
        const bool in_img = lp < tile * tile && px < W && py < H;
        double dir[3] = {0.0, 0.0, 1.0};
        if (in_img) pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
        const float dfx = static_cast<float>(dir[0]), dfy = static_cast<float>(dir[1]),
                    dfz = static_cast<float>(dir[2]);
        const double o0 = a.cam.o[0], o1 = a.cam.o[1], o2 = a.cam.o[2];

        double T = 1.0;
        double acc[3] = {0.0, 0.0, 0.0};
        int32_t k_id[KK];
        double k_w[KK], k_t[KK];
        uint32_t k_seq[KK];
#pragma unroll
        for (int s = 0; s < KK; ++s) {
            k_id[s] = -1;
            k_w[s] = 0.0;
            k_t[s] = 0.0;
            k_seq[s] = 0;
        }
        int k_size = 0;
        uint32_t counter = 0;
        bool active = in_img;
        int dbg_n = 0;
        const bool dbg_row = kDebug && in_img && py >= a.dbg_y0 && py < a.dbg_y1;
        const int64_t dbg_q = kDebug ? (static_cast<int64_t>(py - a.dbg_y0) * W + px) : 0;

        for (int cb = list_begin; cb < list_end; cb += kChunk) {
            const int cn = min(kChunk, list_end - cb);
            __syncthreads();
            for (int e = threadIdx.x; e < cn * 4; e += kThreads) {
                const int j = e >> 2, q = e & 3;
                const int32_t id = __ldg(a.list_ids + cb + j);
                s_f[j][q] = __ldg(a.recf + static_cast<int64_t>(id) * 4 + q);
                if (q == 0) s_id[j] = id;
            }
            for (int e = threadIdx.x; e < cn * kRecPairs; e += kThreads) {
                const int j = e / kRecPairs, q = e - j * kRecPairs;
                const int32_t id = __ldg(a.list_ids + cb + j);
                s_d[j][q] = __ldg(reinterpret_cast<const double2*>(a.rec) + static_cast<int64_t>(id) * kRecPairs + q);
            }
            __syncthreads();
            if (active) {
                // ---- A. prefilter the whole chunk into a survivor mask
                uint32_t m[kChunk / 32];
#pragma unroll
                for (int w = 0; w < kChunk / 32; ++w) {
                    uint32_t bits = 0;
                    const int jn = min(32, cn - 32 * w);
#pragma unroll 4
                    for (int b = 0; b < jn; ++b)
                        if (prefilter(&s_f[32 * w + b][0], dfx, dfy, dfz, near_eps_f)) bits |= 1u << b;
                    m[w] = bits;
                }
                // ---- B. exact fp64 path over this lane's survivors, in list order
#pragma unroll
                for (int w = 0; w < kChunk / 32; ++w) {
                    uint32_t bits = m[w];
                    while (bits && active) {
                        const int j = 32 * w + (__ffs(bits) - 1);
                        bits &= bits - 1;
                        const double* r = reinterpret_cast<const double*>(&s_d[j][0]);
                        // intersect (intersect.hpp:23-42)
                        const double denom = dir[0] * r[REC_NX] + dir[1] * r[REC_NY] + dir[2] * r[REC_NZ];
                        if (fabs(denom) < kMinNormalDot) continue;
                        const double tt = r[REC_NUM] / denom;
                        if (!(tt > near_eps)) continue;
                        const double e0 = (o0 + tt * dir[0]) - r[REC_MUX];
                        const double e1 = (o1 + tt * dir[1]) - r[REC_MUY];
                        const double e2 = (o2 + tt * dir[2]) - r[REC_MUZ];
                        const double du = e0 * r[REC_V1X] + e1 * r[REC_V1Y] + e2 * r[REC_V1Z];
                        if (fabs(du) > r[REC_ULIM]) continue;
                        const double dv = e0 * r[REC_V2X] + e1 * r[REC_V2Y] + e2 * r[REC_V2Z];
                        if (fabs(dv) > r[REC_VLIM]) continue;
                        const double u = du / r[REC_SX];
                        const double v = dv / r[REC_SY];
                        const double alpha_raw = fm::eval_kernel(u, v, r[REC_OP], r[REC_GX], r[REC_GY]);
                        if (alpha_raw < kAlphaMin) continue;
                        // composite (renderer.cpp:146-152)
                        const int32_t id = s_id[j];
                        const double alpha = alpha_max < alpha_raw ? alpha_max : alpha_raw;
                        const double wgt = alpha * T;
                        float col[3];
                        eval_sh_f32(a.sh + static_cast<int64_t>(id) * NX_SH_VALUES, dfx, dfy, dfz, a.sh_degree, col);
                        acc[0] += wgt * col[0];
                        acc[1] += wgt * col[1];
                        acc[2] += wgt * col[2];
                        if (K > 0) {  // TopKBuffer::insert (framebuffers.hpp:33-48)
                            const uint32_t seq = counter++;
                            if (k_size < K) {
#pragma unroll
                                for (int s = 0; s < KK; ++s)
                                    if (s == k_size) {
                                        k_id[s] = id;
                                        k_w[s] = wgt;
                                        k_t[s] = tt;
                                        k_seq[s] = seq;
                                    }
                                ++k_size;
                            } else {
                                // last-ranked incumbent: smallest weight, latest arrival among ties
                                int mi = 0;
                                double wm = k_w[0];
                                uint32_t qm = k_seq[0];
#pragma unroll
                                for (int s = 1; s < KK; ++s)
                                    if (k_w[s] < wm || (k_w[s] == wm && k_seq[s] > qm)) {
                                        mi = s;
                                        wm = k_w[s];
                                        qm = k_seq[s];
                                    }
#pragma unroll
                                for (int s = 0; s < KK; ++s)
                                    if (s == mi && wgt > wm) {
                                        k_id[s] = id;
                                        k_w[s] = wgt;
                                        k_t[s] = tt;
                                        k_seq[s] = seq;
                                    }
                            }
                        }
                        if (kDebug && dbg_row) {
                            if (dbg_n < a.dbg_max) a.dbg_hits[dbg_q * a.dbg_max + dbg_n] = id;
                            ++dbg_n;
                        }
                        T *= 1.0 - alpha;
                        if (T < min_T) active = false;
                    }
                }
            }
            if (!__syncthreads_or(active)) break;
        }

        if (in_img) {
            const int64_t pix = static_cast<int64_t>(py) * W + px;
            a.fb.residual[pix] = static_cast<float>(T);
            acc[0] += T * a.st.background[0];
            acc[1] += T * a.st.background[1];
            acc[2] += T * a.st.background[2];
            if (K > 0) {
                // finalize: weight desc, seq asc (framebuffers.hpp:51-56); slots >= size keep sentinels.
#pragma unroll
                for (int i = 0; i < K; ++i)
#pragma unroll
                    for (int j = 0; j + 1 < K - i; ++j) {
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
                        }
                    }
                // write slots; subtract the buffered primitives' own colours (renderer.cpp:157-164)
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int64_t sl = pix * K + j;
                    a.fb.ids[sl] = k_id[j];
                    a.fb.depths[sl] = k_t[j];
                    a.fb.weights[sl] = k_w[j];
                    if (j < k_size) {
                        float col[3];
                        eval_sh_f32(a.sh + static_cast<int64_t>(k_id[j]) * NX_SH_VALUES, dfx, dfy, dfz, a.sh_degree,
                                    col);
                        acc[0] -= k_w[j] * col[0];
                        acc[1] -= k_w[j] * col[1];
                        acc[2] -= k_w[j] * col[2];
                    }
                }
            }
            a.fb.base[pix * 3 + 0] = static_cast<float>(acc[0]);
            a.fb.base[pix * 3 + 1] = static_cast<float>(acc[1]);
            a.fb.base[pix * 3 + 2] = static_cast<float>(acc[2]);
            if (kDebug && dbg_row) a.dbg_counts[dbg_q] = dbg_n;
        }
    }
}

template <bool kDebug>
void launch_k(const CompositeArgs& a, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(a.fb.tiles_x) * a.fb.tiles_y;
    switch (a.fb.K) {
        case 0: composite_kernel<0, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 1: composite_kernel<1, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 2: composite_kernel<2, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 3: composite_kernel<3, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 4: composite_kernel<4, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 5: composite_kernel<5, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 6: composite_kernel<6, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        case 7: composite_kernel<7, kDebug><<<grid, kThreads, 0, s>>>(a); break;
        default: composite_kernel<8, kDebug><<<grid, kThreads, 0, s>>>(a); break;
    }
}

}  // namespace

void launch_composite(const CompositeArgs& a, cudaStream_t s) {
    count_launch();
    if (a.dbg_hits) launch_k<true>(a, s);
    else launch_k<false>(a, s);
}

}  // namespace nx
