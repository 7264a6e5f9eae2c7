// render_backward (renderer.cpp:251-401) on sm_100a: the compositing branch and
// the per-primitive activation backward. The field branch (field_backward_batch)
// lives in nx_field_backward.cu / nx_field_backward_tc.cu.
//
// Compositing branch (renderer.cpp:287-390). The reference re-marches every pixel
// of every tile front to back, then walks the hits back to front with the suffix
// accumulator A (dL/dw_j * w_j summed behind hit j, seeded by the background
// term). Here one thread per pixel walks the same work lists as the forward
// composite (identical hit sequences: the lists are order-preserving subsequences
// that drop only provable misses) ONCE, front to back, using
//     A_total = dot(dL/dfinal, base) + sum_j dL/dw_j * w_j   (buffered slots j)
// — the fp64 base the forward kept (Eq. 6: the unbuffered colours plus the
// background behind the terminal transmittance) — so that A before hit i is
// A_total minus the running prefix of dL/dw * w. Everything on the geometric
// chain is fp64 with the reference's formulas: eval_kernel_grad (kernel.hpp:
// 40-68), intersect_backward (intersect.hpp:56-87); SH gradients (eval_sh_backward,
// sh.hpp:76-83) are formed in fp32 and accumulated in fp64. The gradient formulas
// multiply by one reciprocal per divisor (values only; every decision stays the
// forward's), and each hit's kernel terms come from its B1 evaluation.
//
// Each warp (8x4 pixels of the work tile) walks the tile's list on its own — its
// own 32-primitive staging, no CTA barriers, so a warp whose pixels terminate early
// stops early. Per group of primitives it pools its survivors like the forward
// (B1: exact fp64 intersect, all lanes busy), composites them per pixel in list
// order (B2: weights, d_alpha, d_t), evaluates every composited pair's gradient (B3a)
// and sums each primitive's per-pixel gradients across the warp in lane order (B3b).
// Those warp sums — the activated gradient (17 values, ActivatedGrad intersect.hpp:
// 45-51), the blended error and the 48 SH gradients — go into per-primitive exact
// accumulators (nx_xacc.cuh), so the result does not depend on the order in which
// warps and tiles meet: render_backward is bit-reproducible, as the reference's is.
// A per-value kernel then reads the accumulators back; activation_backward
// (intersect.hpp:91-103) is linear in the activated gradient, so a final
// per-primitive kernel applies it once to the sum.
#include "nx_fastmath.cuh"
#include "nx_composite.cuh"
#include "nx_xacc.cuh"

namespace nx {

namespace {

// One thread per pixel of the work tile: 8x8 (2 warps of 8x4 pixels, the forward's work
// tiles, so the forward's lists can be reused) or 16x16 (8 warps; NX_BWD_TILE=16).
constexpr int kChunk = 32;                      // primitives staged per warp round
constexpr int kSub = 2;                         // primitives pooled per B1/B2/B3 round
constexpr int kPool = 32 * kSub;
constexpr int kRecPairs = REC_FIELDS / 2;

constexpr int kStage = kActFields + 3;          // per-hit staged values: activated grads, werr, w dL/dfinal

struct BwdHit {         // one evaluated (pixel, primitive) pair
    double alpha;       // B1: raw kernel alpha (< 0: miss); B2: d_alpha
    double t;           // B1: plane crossing
    double d_t;         // B2: upstream dL/dt (field branch) of a buffered hit
    double werr;        // B2: w * err_pixel
    double pu, pv;      // B1: axis_power(u, gx), axis_power(v, gy) (kernel.hpp:16-22)
    double lu, lv;      // B1: log|u|, log|v| (0 for a zero coordinate)
    double k;           // B1: exp(-(pu + pv) / 2)
    float rgb[3];       // B1: primitive colour; B2: w * dL/dfinal * clamp mask (unbuffered), else 0
    uint32_t flags;     // bits 0..2: SH clamp mask (B1)
};
// B3 overwrites a composited entry with its gradient values (float g[kStage]); the
// blended-error term w * err stays fp64 beside it (summed in fp64: the density
// control's split keys depend on it).
struct BwdEntry {
    union {
        BwdHit h;
        float g[kStage + 1];
    };
    double werr64;
};
static_assert(sizeof(BwdHit) <= sizeof(float) * (kStage + 1), "the kernel terms fit the gradient row");
constexpr uint16_t kComposited = 0x80;  // q entry flag set by B2 (list index j < kChunk)

struct WarpSmem {        // one warp's private staging (no sharing between warps)
    float4 f[kChunk][4];
    uint8_t sel[kChunk];     // chunk slots whose support may meet the warp's block (list order)
    uint32_t lmask[kChunk];  // and the block's lanes inside their pixel rects
    float cdir[4][3];        // the block's corner-pixel ray directions (support cull)
    double dir[32][3];
    float basis[32][16];  // per-pixel SH basis (fp32)
    BwdEntry res[kPool];
    int32_t id[kChunk];
    uint16_t q[kPool];
};

// eval_kernel_grad (kernel.hpp:40-68) + intersect_backward (intersect.hpp:56-87):
// the activated-space gradient of one hit, g[0..16] = d_mu[3], d_R[9] (m[i][j]),
// d_sigma[2], d_opacity, d_gamma[2]. The kernel terms (axis powers, log|u|, log|v|,
// exp(-(pu + pv)/2)) are the ones B1 formed for the hit (finite: a composited hit).
__device__ __forceinline__ void hit_backward(const double* r, const double* d, const double* o, double t, double u,
                                             double v, double rsx, double rsy, const BwdHit& hh, double* g) {
    const double op = r[REC_OP], gx = r[REC_GX], gy = r[REC_GY];
    const double pu = hh.pu, pv = hh.pv, d_alpha = hh.alpha, d_t = hh.d_t;
    double kd_u = 0.0, kd_v = 0.0, kd_gx = 0.0, kd_gy = 0.0;
    const double k = hh.k;
    const double alpha = op * k;
    const double kd_op = k;
    if (u != 0.0) {
        const double au = fabs(u);
        kd_u = -alpha * gx * (pu / au) * (u > 0 ? 1.0 : -1.0);
        kd_gx = -alpha * hh.lu * pu;
    }
    if (v != 0.0) {
        const double av = fabs(v);
        kd_v = -alpha * gy * (pv / av) * (v > 0 ? 1.0 : -1.0);
        kd_gy = -alpha * hh.lv * pv;
    }
    const double v1[3] = {r[REC_V1X], r[REC_V1Y], r[REC_V1Z]};
    const double v2[3] = {r[REC_V2X], r[REC_V2Y], r[REC_V2Z]};
    const double n[3] = {r[REC_NX], r[REC_NY], r[REC_NZ]};
    const double mu[3] = {r[REC_MUX], r[REC_MUY], r[REC_MUZ]};
    const double denom = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
    const double x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    // gradient values only (no decision depends on them): one reciprocal per divisor
    // instead of the reference's nine divisions
    const double rden = 1.0 / denom;
    g[14] = d_alpha * kd_op;
    g[15] = d_alpha * kd_gx;
    g[16] = d_alpha * kd_gy;
    g[12] = d_alpha * kd_u * (-u * rsx);
    g[13] = d_alpha * kd_v * (-v * rsy);
    const double du = d_alpha * kd_u, dv = d_alpha * kd_v;
    const double dv1 = d[0] * v1[0] + d[1] * v1[1] + d[2] * v1[2];
    const double dv2 = d[0] * v2[0] + d[1] * v2[1] + d[2] * v2[2];
    const double au = du * rsx, av = dv * rsy;
    const double dt = d_t + au * dv1 + av * dv2;
    const double cu = -au, cv = -av, cn = dt * rden;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        g[i] = cu * v1[i] + cv * v2[i] + cn * n[i];
        const double xm = x[i] - mu[i];
        g[3 + 3 * i + 0] = au * xm;
        g[3 + 3 * i + 1] = av * xm;
        g[3 + 3 * i + 2] = cn * (-xm);
    }
}

template <int K, int kTile>
__global__ void __launch_bounds__(kTile * kTile, 512 / (kTile * kTile)) composite_bwd_kernel(const CompositeBwdArgs a) {
    constexpr int KK = K > 0 ? K : 1;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];

    const int t = blockIdx.x;
    const int tx = t % a.fb.tiles_x, ty = t / a.fb.tiles_x;
    const int list_begin = a.tile_offsets[t], list_end = a.tile_offsets[t + 1];
    const int W = a.cam.W, H = a.cam.H;
    const double near_eps = a.st.near_eps, alpha_max = a.st.alpha_max, min_T = a.st.min_transmittance;
    const float near_eps_f = static_cast<float>(near_eps);
    const double o[3] = {a.cam.o[0], a.cam.o[1], a.cam.o[2]};

    // warp w owns the 8x4 block (w % (kTile / 8), w / (kTile / 8)) of the tile
    constexpr int kAcross = kTile / 8;
    const int px = tx * kTile + (warp % kAcross) * 8 + (lane & 7), py = ty * kTile + (warp / kAcross) * 4 + (lane >> 3);
    const bool in_img = px < W && py < H;
    const int wx0 = __reduce_min_sync(0xffffffffu, in_img ? px : 0x7fffffff);
    const int wx1 = __reduce_max_sync(0xffffffffu, in_img ? px : -1);
    const int wy0 = __reduce_min_sync(0xffffffffu, in_img ? py : 0x7fffffff);
    const int wy1 = __reduce_max_sync(0xffffffffu, in_img ? py : -1);
    double dir[3] = {0.0, 0.0, 1.0};
    if (in_img) pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
    sm.dir[lane][0] = dir[0];
    sm.dir[lane][1] = dir[1];
    sm.dir[lane][2] = dir[2];
    const float dfx = static_cast<float>(dir[0]), dfy = static_cast<float>(dir[1]), dfz = static_cast<float>(dir[2]);
    sh_basis_f32(dfx, dfy, dfz, sm.basis[lane]);
    // the block's corner pixels (lanes 0, 7, 24, 31) for the support cull (as the forward)
    const uint32_t in_mask = __ballot_sync(0xffffffffu, in_img);
    constexpr uint32_t kCorners = (1u << 0) | (1u << 7) | (1u << 24) | (1u << 31);
    const bool quad_ok = (in_mask & kCorners) == kCorners;
    {
        const int ci = lane == 0 ? 0 : lane == 7 ? 1 : lane == 24 ? 2 : lane == 31 ? 3 : -1;
        if (ci >= 0) {
            sm.cdir[ci][0] = dfx;
            sm.cdir[ci][1] = dfy;
            sm.cdir[ci][2] = dfz;
        }
    }
    const int bx0 = tx * kTile + (warp % kAcross) * 8, by0 = ty * kTile + (warp / kAcross) * 4;

    // per-pixel upstream state
    const int64_t pix = in_img ? static_cast<int64_t>(py) * W + px : 0;
    double dfin[3] = {0.0, 0.0, 0.0};
    if (in_img && a.d_final)
        for (int c = 0; c < 3; ++c) dfin[c] = a.d_final[pix * 3 + c];
    int32_t k_id[KK];
    double k_dw[KK], k_dt[KK];
    double A_total = 0.0;
#pragma unroll
    for (int j = 0; j < KK; ++j) {
        k_id[j] = -1;
        k_dw[j] = 0.0;
        k_dt[j] = 0.0;
    }
    if (in_img) {
        A_total = dfin[0] * a.fb.base64[pix * 3 + 0] + dfin[1] * a.fb.base64[pix * 3 + 1] +
                  dfin[2] * a.fb.base64[pix * 3 + 2];
        if (K > 0) {
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                const int64_t sl = pix * K + j;
                k_id[j] = a.fb.ids[sl];
                if (k_id[j] < 0) continue;
                const float* tex = a.fb.texture + sl * 3;
                double dw = dfin[0] * tex[0] + dfin[1] * tex[1] + dfin[2] * tex[2];  // dot(dfin, tex)
                if (a.d_weights) dw += a.d_weights[sl];
                k_dw[j] = dw;
                k_dt[j] = a.d_t_slot[sl];
                A_total += dw * a.fb.weights[sl];
            }
        }
    }
    const double errp = (in_img && a.err_pixel) ? a.err_pixel[pix] : 0.0;
    const int n_act = a.err_pixel ? kActFields : kActFields - 1;
    const int n_sh = a.sh_degree >= 3 ? 16 : 1;
    const Xacc acc = a.acc;

    double T = 1.0, P = 0.0;
    bool active = in_img;
    const double2* rec2 = reinterpret_cast<const double2*>(a.rec);

    for (int cb = list_begin; cb < list_end; cb += kChunk) {
        if (!__any_sync(0xffffffffu, active)) break;
        const int cn = min(kChunk, list_end - cb);
        __syncwarp();
        if (lane < cn) {  // the prefilter records, gathered by id, with cp.async (as the forward)
            const int32_t id = __ldg(a.list_ids + cb + lane);
            sm.id[lane] = id;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&sm.f[lane][q]));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                             "l"(a.recf + static_cast<int64_t>(id) * 4 + q)
                             : "memory");
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        // the chunk's primitives whose support may meet this warp's block, in list order:
        // pixel rect overlap, then the corner-ray quadrilateral (nx_composite.cu)
        int nsel = 0;
        {
            bool ov = false;
            uint32_t lm = 0;
            if (lane < cn) {
                const float4 f3 = sm.f[lane][3];
                const int rx = __float_as_int(f3.z), ry = __float_as_int(f3.w);
                ov = !((rx >> 16) < wx0 || (rx & 0xffff) > wx1 || (ry >> 16) < wy0 || (ry & 0xffff) > wy1);
                if (ov && quad_ok) {
                    const float4 f0 = sm.f[lane][0], f1 = sm.f[lane][1], f2 = sm.f[lane][2];
                    float umin = 3e38f, umax = -3e38f, vmin = 3e38f, vmax = -3e38f, su = 0.f, sv = 0.f, sgn = 0.f;
                    bool valid = true;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float dx = sm.cdir[c][0], dy = sm.cdir[c][1], dz = sm.cdir[c][2];
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
                if (ov) {
                    const int cx0 = max((rx & 0xffff) - bx0, 0), cx1 = min((rx >> 16) - bx0, 7);
                    const int ry0 = max((ry & 0xffff) - by0, 0), ry1 = min((ry >> 16) - by0, 3);
                    const uint32_t cols = (0xffu >> (7 - cx1)) & (0xffu << cx0);
                    const uint32_t rows = (0xffffffffu >> (8 * (3 - ry1))) & (0xffffffffu << (8 * ry0));
                    lm = (cols * 0x01010101u) & rows;
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, ov);
            if (ov) {
                const int slot = __popc(m & ((1u << lane) - 1u));
                sm.sel[slot] = static_cast<uint8_t>(lane);
                sm.lmask[slot] = lm;
            }
            nsel = __popc(m);
        }
        __syncwarp();
        for (int g0 = 0; g0 < nsel; g0 += kSub) {
            const int gn = min(kSub, nsel - g0);
            // ---- A. pixel rect (lane mask) + fp32 prefilter (as the forward)
            uint32_t mask = 0;
#pragma unroll
            for (int b = 0; b < kSub; ++b) {
                if (b >= gn) break;
                const int j = sm.sel[g0 + b];
                if (active && ((sm.lmask[g0 + b] >> lane) & 1u) && prefilter(&sm.f[j][0], dfx, dfy, dfz, near_eps_f))
                    mask |= 1u << b;
            }
            const int cnt = __popc(mask);
            int incl = cnt;
#pragma unroll
            for (int of = 1; of < 32; of <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, of);
                if (lane >= of) incl += y;
            }
            const int off = incl - cnt;
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) continue;
            {
                uint32_t m = mask;
                int k = off;
                while (m) {
                    const int b = __ffs(m) - 1;
                    m &= m - 1;
                    sm.q[k++] = static_cast<uint16_t>((lane << 8) | sm.sel[g0 + b]);
                }
            }
            __syncwarp();
            // ---- B1. exact fp64 intersect of the pooled pairs (intersect.hpp:23-42)
            for (int e = lane; e < total; e += 32) {
                const int ent = sm.q[e];
                const int owner = ent >> 8, j = ent & 0x7f;
                const double d0 = sm.dir[owner][0], d1 = sm.dir[owner][1], d2 = sm.dir[owner][2];
                const int32_t id = sm.id[j];
                double r[REC_FIELDS];
#pragma unroll
                for (int q = 0; q < kRecPairs; ++q) {
                    const double2 v = __ldg(rec2 + static_cast<int64_t>(id) * kRecPairs + q);
                    r[2 * q] = v.x;
                    r[2 * q + 1] = v.y;
                }
                BwdHit res;
                res.alpha = -1.0;
                res.t = 0.0;
                res.flags = 0;
                // intersect + eval_kernel, keeping the kernel terms for B3a (the forward's
                // exact_hit, so both passes take the same decisions)
                const HitTerms h = exact_hit(r, d0, d1, d2, o[0], o[1], o[2], near_eps);
                if (h.alpha >= 0.0) {
                    res.alpha = h.alpha;
                    res.t = h.t;
                    res.pu = h.pu;
                    res.pv = h.pv;
                    res.lu = h.lu;
                    res.lv = h.lv;
                    res.k = h.k;
                    uint32_t act;
                    eval_sh_f32(a.sh + static_cast<int64_t>(id) * NX_SH_VALUES, static_cast<float>(d0),
                                static_cast<float>(d1), static_cast<float>(d2), a.sh_degree, res.rgb, &act);
                    res.flags = act;
                }
                sm.res[e].h = res;
            }
            __syncwarp();
            // ---- B2. per-pixel march in list order: weights, d_alpha, d_t (renderer.cpp:325-370)
            for (int k = off; k < off + cnt && active; ++k) {
                BwdHit& res = sm.res[k].h;
                if (res.alpha < 0.0) continue;
                const int32_t id = sm.id[sm.q[k] & 0x7f];
                const bool clamped = res.alpha > alpha_max;
                const double alpha = clamped ? alpha_max : res.alpha;
                const double w = alpha * T;
                int slot = -1;
#pragma unroll
                for (int j = 0; j < KK; ++j)
                    if (K > 0 && slot < 0 && k_id[j] == id) slot = j;
                double dw = 0.0, d_t = 0.0;
                float wdf[3] = {0.f, 0.f, 0.f};
                if (slot >= 0) {
#pragma unroll
                    for (int j = 0; j < KK; ++j)
                        if (j == slot) {
                            dw = k_dw[j];
                            d_t = k_dt[j];
                        }
                } else {
                    dw = dfin[0] * res.rgb[0] + dfin[1] * res.rgb[1] + dfin[2] * res.rgb[2];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        wdf[c] = (res.flags >> c) & 1u ? static_cast<float>(w * dfin[c]) : 0.f;
                }
                const double A = A_total - P - dw * w;  // sum of dL/dw * w behind this hit
                double d_alpha = dw * T - A / (1.0 - alpha);
                if (clamped) d_alpha = 0.0;
                P += dw * w;
                res.alpha = d_alpha;
                res.d_t = d_t;
                res.werr = w * errp;
                sm.res[k].werr64 = res.werr;
                res.rgb[0] = wdf[0];
                res.rgb[1] = wdf[1];
                res.rgb[2] = wdf[2];
                sm.q[k] |= kComposited;
                T *= 1.0 - alpha;
                if (T < min_T) active = false;
            }
            __syncwarp();
            // ---- B3a. gradients of every composited pair, all lanes busy: eval_kernel_grad +
            // intersect_backward in fp64 -> staged as fp32 in the entry
#pragma unroll 1
            for (int e = lane; e < total; e += 32) {
                const int ent = sm.q[e];
                if (!(ent & kComposited)) continue;
                const BwdHit hh = sm.res[e].h;
                const int owner = ent >> 8;
                const double d3[3] = {sm.dir[owner][0], sm.dir[owner][1], sm.dir[owner][2]};
                const int32_t id = sm.id[ent & 0x7f];
                double r[REC_FIELDS];
#pragma unroll
                for (int q = 0; q < kRecPairs; ++q) {
                    const double2 v = __ldg(rec2 + static_cast<int64_t>(id) * kRecPairs + q);
                    r[2 * q] = v.x;
                    r[2 * q + 1] = v.y;
                }
                // the hit's plane coordinates, as intersect() formed them
                const double e0 = (o[0] + hh.t * d3[0]) - r[REC_MUX];
                const double e1 = (o[1] + hh.t * d3[1]) - r[REC_MUY];
                const double e2 = (o[2] + hh.t * d3[2]) - r[REC_MUZ];
                const double rsx = 1.0 / r[REC_SX], rsy = 1.0 / r[REC_SY];
                const double u = (e0 * r[REC_V1X] + e1 * r[REC_V1Y] + e2 * r[REC_V1Z]) * rsx;
                const double v = (e0 * r[REC_V2X] + e1 * r[REC_V2Y] + e2 * r[REC_V2Z]) * rsy;
                double gd[kActFields - 1];
                hit_backward(r, d3, o, hh.t, u, v, rsx, rsy, hh, gd);
                float* g = sm.res[e].g;
#pragma unroll
                for (int i = 0; i < kActFields - 1; ++i) g[i] = static_cast<float>(gd[i]);
                g[kActFields - 1] = static_cast<float>(hh.werr);
                g[kActFields + 0] = hh.rgb[0];
                g[kActFields + 1] = hh.rgb[1];
                g[kActFields + 2] = hh.rgb[2];
            }
            __syncwarp();
            // ---- B3b. per primitive of the group, one pass over the pixels that hit it (lane
            // order): lanes 0..15 sum the SH gradients of coefficient k = lane for the three
            // channels (w dL/dfinal x basis_k of the pixel), lanes 16..31 the activated values
            // lane - 16 (and lanes 16, 17 also values 16, 17); the warp sums go into the
            // primitive's exact accumulators
            int cur = off;
            const bool sh_lane = lane < 16;
            const int av = lane - 16;  // activated value of an act lane (and av + 16 for lanes 16, 17)
#pragma unroll 1
            for (int b = 0; b < gn; ++b) {
                const int j = sm.sel[g0 + b];
                int my_e = -1;
                if (cur < off + cnt && (sm.q[cur] & 0x7f) == j) {
                    if (sm.q[cur] & kComposited) my_e = cur;
                    ++cur;
                }
                const uint32_t hm = __ballot_sync(0xffffffffu, my_e >= 0);
                if (!hm) continue;
                const int64_t row = static_cast<int64_t>(sm.id[j]) * kPrimAccVals;
                // the blended error in fp64: a fixed-pattern warp tree over the pixels' terms
                double werr = my_e >= 0 ? sm.res[my_e].werr64 : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) werr += __shfl_xor_sync(0xffffffffu, werr, o);
                float s0 = 0.f, s1 = 0.f, s2 = 0.f;
                for (uint32_t m = hm; m; m &= m - 1) {
                    const int h = __ffs(m) - 1;
                    const int eh = __shfl_sync(0xffffffffu, my_e, h);
                    const float* g = sm.res[eh].g;
                    if (sh_lane) {
                        const float bk = sm.basis[h][lane];
                        s0 = fmaf(g[kActFields + 0], bk, s0);
                        s1 = fmaf(g[kActFields + 1], bk, s1);
                        s2 = fmaf(g[kActFields + 2], bk, s2);
                    } else {
                        s0 += g[av];
                        if (av < kActFields - 16) s1 += g[av + 16];
                    }
                }
                if (sh_lane) {
                    if (lane < n_sh) {
                        const int64_t base = row + kActFields + 3 * lane;
                        if (s0 != 0.f) xacc_add(acc, base + 0, s0);
                        if (s1 != 0.f) xacc_add(acc, base + 1, s1);
                        if (s2 != 0.f) xacc_add(acc, base + 2, s2);
                    }
                } else {
                    if (s0 != 0.f && av < n_act) xacc_add(acc, row + av, s0);
                    if (av == 0 && s1 != 0.f) xacc_add(acc, row + 16, s1);
                    if (av == 1 && werr != 0.0 && 17 < n_act) xacc_add(acc, row + 17, werr);
                }
            }
            __syncwarp();
        }
    }
}

template <int K>
void launch_one(const CompositeBwdArgs& a, unsigned grid, cudaStream_t s) {
    if (a.tile == 8) {
        const size_t smem = 2 * sizeof(WarpSmem);
        cudaFuncSetAttribute(composite_bwd_kernel<K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        composite_bwd_kernel<K, 8><<<grid, 64, smem, s>>>(a);
    } else {
        const size_t smem = 8 * sizeof(WarpSmem);
        cudaFuncSetAttribute(composite_bwd_kernel<K, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        composite_bwd_kernel<K, 16><<<grid, 256, smem, s>>>(a);
    }
}

// quat_rotation_backward (primitive.cpp:22-45)
__device__ void quat_rotation_backward(const double* q_raw, const double* g, double* dq) {
    const double n = sqrt(q_raw[0] * q_raw[0] + q_raw[1] * q_raw[1] + q_raw[2] * q_raw[2] + q_raw[3] * q_raw[3]);
    const double inv = 1.0 / n;
    const double w = inv * q_raw[0], x = inv * q_raw[1], y = inv * q_raw[2], z = inv * q_raw[3];
    // g[3*i + j] = d_R.m[i][j]
    double du[4];
    du[0] = 2 * (-z * g[1] + y * g[2] + z * g[3] - x * g[5] - y * g[6] + x * g[7]);
    du[1] = 2 * (y * g[1] + z * g[2] + y * g[3] - 2 * x * g[4] - w * g[5] + z * g[6] + w * g[7] - 2 * x * g[8]);
    du[2] = 2 * (-2 * y * g[0] + x * g[1] + w * g[2] + x * g[3] + z * g[5] - w * g[6] + z * g[7] - 2 * y * g[8]);
    du[3] = 2 * (-2 * z * g[0] - w * g[1] + x * g[2] + w * g[3] - 2 * z * g[4] + y * g[5] + x * g[6] + y * g[7]);
    const double u[4] = {w, x, y, z};
    const double r = du[0] * u[0] + du[1] * u[1] + du[2] * u[2] + du[3] * u[3];
    for (int k = 0; k < 4; ++k) dq[k] = (du[k] - r * u[k]) / n;
}

// Reads the exact per-primitive sums back (zeroing them): the activated part into
// act_grad for prim_finalize_kernel, the SH part added to PrimitiveGrad.
__global__ void prim_take_kernel(const Xacc acc, int64_t n, double* __restrict__ act_grad,
                                 double* __restrict__ prim_grad) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * kPrimAccVals) return;
    const int64_t i = idx / kPrimAccVals;
    const int v = static_cast<int>(idx - i * kPrimAccVals);
    const double val = xacc_take(acc, idx);
    if (v < kActFields) act_grad[i * kActFields + v] = val;
    else if (val != 0.0) prim_grad[i * NX_PARAMS_PER_NEXEL + 12 + (v - kActFields)] += val;
}

// activation_backward (intersect.hpp:91-103) applied to the per-primitive sum of the
// activated gradients (it is linear in them), + the blended-error sum.
__global__ void prim_finalize_kernel(const SceneDev scene, int no_gamma, const double* __restrict__ act_grad,
                                     double* __restrict__ prim_grad, double* __restrict__ blended_error) {
    const int64_t n = scene.n;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double g[kActFields];
    bool any = false;
#pragma unroll
    for (int k = 0; k < kActFields; ++k) {
        g[k] = act_grad[i * kActFields + k];
        any |= g[k] != 0.0;
    }
    if (!any) return;
    const double* geo = scene.geom;
    double* out = prim_grad + i * NX_PARAMS_PER_NEXEL;
    out[0] += g[0];
    out[1] += g[1];
    out[2] += g[2];
    const double q[4] = {geo[3 * n + i], geo[4 * n + i], geo[5 * n + i], geo[6 * n + i]};
    double dq[4];
    quat_rotation_backward(q, g + 3, dq);
    for (int k = 0; k < 4; ++k) out[3 + k] += dq[k];
    out[7] += g[12] * exp(geo[7 * n + i]);
    out[8] += g[13] * exp(geo[8 * n + i]);
    const double op = sigmoid(geo[9 * n + i]);
    out[9] += g[14] * op * (1.0 - op);
    if (!no_gamma) {
        out[10] += g[15] * sigmoid(geo[10 * n + i]);  // softplus_grad (vec_math.hpp:87)
        out[11] += g[16] * sigmoid(geo[11 * n + i]);
    }
    if (blended_error) blended_error[i] += g[17];
}

}  // namespace

void launch_composite_backward(const CompositeBwdArgs& a, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>(a.fb.tiles_x) * a.fb.tiles_y;
    if (grid == 0) return;
    count_launch();
    switch (a.fb.K) {
        case 0: launch_one<0>(a, grid, s); break;
        case 1: launch_one<1>(a, grid, s); break;
        case 2: launch_one<2>(a, grid, s); break;
        case 3: launch_one<3>(a, grid, s); break;
        case 4: launch_one<4>(a, grid, s); break;
        case 5: launch_one<5>(a, grid, s); break;
        case 6: launch_one<6>(a, grid, s); break;
        case 7: launch_one<7>(a, grid, s); break;
        default: launch_one<8>(a, grid, s); break;
    }
}

void launch_prim_finalize(const SceneDev& scene, int no_gamma, const Xacc& acc, double* act_grad, double* prim_grad,
                          double* blended_error, cudaStream_t s) {
    if (scene.n <= 0) return;
    count_launch();
    const int64_t nv = scene.n * kPrimAccVals;
    prim_take_kernel<<<static_cast<unsigned>((nv + 255) / 256), 256, 0, s>>>(acc, scene.n, act_grad, prim_grad);
    count_launch();
    prim_finalize_kernel<<<static_cast<unsigned>((scene.n + 255) / 256), 256, 0, s>>>(scene, no_gamma, act_grad,
                                                                                     prim_grad, blended_error);
}

}  // namespace nx
