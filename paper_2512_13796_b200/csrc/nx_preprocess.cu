// K1 preprocess + binning helpers.
//
// One thread per primitive, fp64 throughout. Restates, per primitive, the
// first half of build_binning (renderer.cpp:52-100): activate (primitive.cpp:
// 47-76), support radius (kernel.hpp:72-76), the four support corners, the
// all_behind / all_visible classification, the centre depth and the padded
// tile rect. It also emits the per-camera composite record and, for the
// straddlers the reference bins into every tile (renderer.cpp:93-98), a
// conservative "work rect" that provably contains every pixel whose ray can hit
// the primitive: the work lists are order-preserving
// subsequences of the reference lists that drop only provable misses.
#include <algorithm>

#include "nx_internal.cuh"

namespace nx {

namespace {

struct D3 {
    double x, y, z;
};

__device__ __forceinline__ D3 to_camera(const CamD& c, D3 p) {  // camera.hpp:26
    return {c.R[0] * p.x + c.R[1] * p.y + c.R[2] * p.z + c.t[0],
            c.R[3] * p.x + c.R[4] * p.y + c.R[5] * p.z + c.t[1],
            c.R[6] * p.x + c.R[7] * p.y + c.R[8] * p.z + c.t[2]};
}

__device__ __forceinline__ int4 empty_rect() { return make_int4(1, 0, 1, 0); }

__device__ __forceinline__ int rect_tiles(int4 r) {
    return (r.y >= r.x && r.w >= r.z) ? (r.y - r.x + 1) * (r.w - r.z + 1) : 0;
}

// Conservative work rect of a straddler: clip the support rectangle (radii padded
// by 1e-6) to camera-z >= zmin, project the clipped polygon, take its bounding box
// padded by 2 px, and convert to tiles. Every hit has t > near_eps, hence
// camera-z > near_eps * cos(ray, axis) >= 2*zmin, and alpha >= 1/255 implies
// |u| <= ru, |v| <= rv (kernel.hpp:70-76).
__device__ int4 straddler_pixel_rect(const CamD& cam, D3 mu, D3 a1, D3 a2, double zmin) {
    D3 poly[8];
    const D3 c0 = to_camera(cam, {mu.x + a1.x + a2.x, mu.y + a1.y + a2.y, mu.z + a1.z + a2.z});
    const D3 c1 = to_camera(cam, {mu.x + a1.x - a2.x, mu.y + a1.y - a2.y, mu.z + a1.z - a2.z});
    const D3 c2 = to_camera(cam, {mu.x - a1.x - a2.x, mu.y - a1.y - a2.y, mu.z - a1.z - a2.z});
    const D3 c3 = to_camera(cam, {mu.x - a1.x + a2.x, mu.y - a1.y + a2.y, mu.z - a1.z + a2.z});
    const D3 in[4] = {c0, c1, c2, c3};
    int m = 0;
    for (int k = 0; k < 4; ++k) {  // Sutherland-Hodgman against z >= zmin
        const D3 a = in[k], b = in[(k + 1) & 3];
        const bool ia = a.z >= zmin, ib = b.z >= zmin;
        if (ia) poly[m++] = a;
        if (ia != ib) {
            const double s = (zmin - a.z) / (b.z - a.z);
            poly[m++] = {a.x + s * (b.x - a.x), a.y + s * (b.y - a.y), zmin};
        }
    }
    if (m == 0) return empty_rect();
    double px0 = 1e300, px1 = -1e300, py0 = 1e300, py1 = -1e300;
    for (int k = 0; k < m; ++k) {
        const double z = fmax(poly[k].z, zmin);
        const double x = cam.fx * poly[k].x / z + cam.cx;
        const double y = cam.fy * poly[k].y / z + cam.cy;
        px0 = fmin(px0, x);
        px1 = fmax(px1, x);
        py0 = fmin(py0, y);
        py1 = fmax(py1, y);
    }
    // pixel i has its centre at i + 0.5; pad 2 px on each side.
    px0 = fmax(px0 - 2.5, -1.0);
    py0 = fmax(py0 - 2.5, -1.0);
    px1 = fmin(px1 + 1.5, static_cast<double>(cam.W) + 1.0);
    py1 = fmin(py1 + 1.5, static_cast<double>(cam.H) + 1.0);
    const int ix0 = static_cast<int>(floor(px0)), ix1 = static_cast<int>(ceil(px1));
    const int iy0 = static_cast<int>(floor(py0)), iy1 = static_cast<int>(ceil(py1));
    if (ix1 < 0 || iy1 < 0 || ix0 >= cam.W || iy0 >= cam.H || ix1 < ix0 || iy1 < iy0) return empty_rect();
    return make_int4(clampi(ix0, 0, cam.W - 1), clampi(ix1, 0, cam.W - 1), clampi(iy0, 0, cam.H - 1),
                     clampi(iy1, 0, cam.H - 1));
}

__device__ __forceinline__ int4 pixel_to_tiles(int4 p, int tile) {
    return p.y >= p.x ? make_int4(p.x / tile, p.y / tile, p.z / tile, p.w / tile) : empty_rect();
}

#ifndef NX_PRE_THREADS
#define NX_PRE_THREADS 256
#endif
#ifndef NX_PRE_MINB
#define NX_PRE_MINB 3  // 80 registers: 3 CTAs of 256 per SM (measured 0.083 -> 0.070 ms at config 2)
#endif
constexpr int kPreThreads = NX_PRE_THREADS;

__global__ void __launch_bounds__(kPreThreads, NX_PRE_MINB) preprocess_kernel(const PreprocessArgs a) {
    __shared__ unsigned long long s_cnt[8];
    if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t n = a.scene.n;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int cls = -1, kept = 0;
    long long ref_keys = 0, work_keys = 0;
    if (i < n) {
        const double* g = a.scene.geom;
        const D3 mu{g[0 * n + i], g[1 * n + i], g[2 * n + i]};
        const double qw = g[3 * n + i], qx = g[4 * n + i], qy = g[5 * n + i], qz = g[6 * n + i];
        // activate (primitive.cpp:62-75); inputs were validated at upload.
        const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
        const double inv = 1.0 / qn;
        const double w = inv * qw, x = inv * qx, y = inv * qy, z = inv * qz;
        double R[9];  // quat_to_rotation (primitive.cpp:7-20)
        R[0] = 1 - 2 * (y * y + z * z);
        R[1] = 2 * (x * y - w * z);
        R[2] = 2 * (x * z + w * y);
        R[3] = 2 * (x * y + w * z);
        R[4] = 1 - 2 * (x * x + z * z);
        R[5] = 2 * (y * z - w * x);
        R[6] = 2 * (x * z - w * y);
        R[7] = 2 * (y * z + w * x);
        R[8] = 1 - 2 * (x * x + y * y);
        const double sx = exp(g[7 * n + i]), sy = exp(g[8 * n + i]);
        const double op = sigmoid(g[9 * n + i]);
        double gx = 1.0, gy = 1.0;
        if (!a.st.no_gamma) {
            gx = 1.0 + softplus(g[10 * n + i]);
            gy = 1.0 + softplus(g[11 * n + i]);
        }
        const double ru = support_radius(op, gx), rv = support_radius(op, gy);
        {  // near-threshold: support radius sign (kernel.hpp:72-76)
            const double lim = 2.0 * log(op / kAlphaMin);
            if (fabs(lim) < kNearSupport) atomicAdd(&a.stats->near[NEAR_SUPPORT], 1ull);
        }
        int4 ref = empty_rect(), work = empty_rect();
        double depth = 0.0;
        int4 prect = empty_rect();  // pixel rect containing every possible hit (work mode)
        if (ru <= 0.0 || rv <= 0.0) {
            cls = CLS_SUPPORT;
        } else {
            const double ku = ru * sx, kv = rv * sy;
            const D3 du{ku * R[0], ku * R[3], ku * R[6]};
            const D3 dv{kv * R[1], kv * R[4], kv * R[7]};
            const D3 corners[4] = {
                {(mu.x + du.x) + dv.x, (mu.y + du.y) + dv.y, (mu.z + du.z) + dv.z},
                {(mu.x + du.x) - dv.x, (mu.y + du.y) - dv.y, (mu.z + du.z) - dv.z},
                {(mu.x - du.x) + dv.x, (mu.y - du.y) + dv.y, (mu.z - du.z) + dv.z},
                {(mu.x - du.x) - dv.x, (mu.y - du.y) - dv.y, (mu.z - du.z) - dv.z}};
            const D3 cmu = to_camera(a.cam, mu);
            bool all_behind = cmu.z < kProjectMinDepth;
            bool all_visible = true;
            double px0 = 1e300, px1 = -1e300, py0 = 1e300, py1 = -1e300;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const D3 q = to_camera(a.cam, corners[c]);
                if (q.z < kProjectMinDepth) {  // camera.hpp:38-42
                    all_visible = false;
                    continue;
                }
                all_behind = false;
                const double X = a.cam.fx * q.x / q.z + a.cam.cx;
                const double Y = a.cam.fy * q.y / q.z + a.cam.cy;
                px0 = X < px0 ? X : px0;  // std::min / std::max (renderer.cpp:71-74)
                px1 = px1 < X ? X : px1;
                py0 = Y < py0 ? Y : py0;
                py1 = py1 < Y ? Y : py1;
            }
            depth = cmu.z;
            if (all_behind && !all_visible) {
                cls = CLS_BEHIND;
            } else if (all_visible) {
                {  // near-threshold: the rect's floor / ceil arguments next to an integer
                    const double v[4] = {px0 - 1.5, px1 + 0.5, py0 - 1.5, py1 + 0.5};
                    int near = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) near |= fabs(v[q] - rint(v[q])) < kNearPixel;
                    if (near) atomicAdd(&a.stats->near[NEAR_RECT], 1ull);
                }
                const int ix0 = x86_to_int(floor(px0 - 1.5)), ix1 = x86_to_int(ceil(px1 + 0.5));
                const int iy0 = x86_to_int(floor(py0 - 1.5)), iy1 = x86_to_int(ceil(py1 + 0.5));
                if (ix1 < 0 || iy1 < 0 || ix0 >= a.cam.W || iy0 >= a.cam.H) {
                    cls = CLS_OFFSCREEN;
                } else {
                    cls = CLS_RECT;
                    // The padded pixel rect contains every pixel centre inside the projected
                    // support quad (all corners in front: the projection is that quad).
                    prect = make_int4(clampi(ix0, 0, a.cam.W - 1), clampi(ix1, 0, a.cam.W - 1),
                                      clampi(iy0, 0, a.cam.H - 1), clampi(iy1, 0, a.cam.H - 1));
                    ref = pixel_to_tiles(prect, a.st.tile);
                    work = pixel_to_tiles(prect, a.work_tile);
                }
            } else {
                cls = CLS_STRADDLER;
                ref = make_int4(0, a.tiles_x - 1, 0, a.tiles_y - 1);
                const double pu = ku * (1.0 + 1e-6), pv = kv * (1.0 + 1e-6);
                prect = straddler_pixel_rect(a.cam, mu, {pu * R[0], pu * R[3], pu * R[6]},
                                             {pv * R[1], pv * R[4], pv * R[7]}, a.zmin_work);
                // Degenerate near-threshold opacity: keep the reference's all-tile list.
                if (log(op / kAlphaMin) < 1e-3) prect = make_int4(0, a.cam.W - 1, 0, a.cam.H - 1);
                work = pixel_to_tiles(prect, a.work_tile);
                kept = rect_tiles(work) > 0;
            }
        }
        if (a.reference_lists) {
            work = (cls == CLS_RECT || cls == CLS_STRADDLER) ? ref : empty_rect();
            prect = make_int4(0, a.cam.W - 1, 0, a.cam.H - 1);  // reference walk: no culling
        }
        a.cls[i] = cls;
        a.ref_rect[i] = ref;
        a.work_rect[i] = work;
        a.key[i] = depth_key(depth);
        const int wk = rect_tiles(work);
        a.flag[i] = wk > 0;
        ref_keys = rect_tiles(ref);
        work_keys = wk;
        if (wk > 0) {
            // Composite records: everything intersect() (intersect.hpp:23-42) needs per
            // primitive (fp64, exact path) + the fp32 prefilter record.
            double r[REC_FIELDS];
            const double nx_ = R[2], ny_ = R[5], nz_ = R[8];
            const double mx = mu.x - a.cam.o[0], my = mu.y - a.cam.o[1], mz = mu.z - a.cam.o[2];
            r[REC_NUM] = mx * nx_ + my * ny_ + mz * nz_;  // dot(a.mu - ray.origin, n)
            r[REC_NX] = nx_;
            r[REC_NY] = ny_;
            r[REC_NZ] = nz_;
            r[REC_V1X] = R[0];
            r[REC_V1Y] = R[3];
            r[REC_V1Z] = R[6];
            r[REC_V2X] = R[1];
            r[REC_V2Y] = R[4];
            r[REC_V2Z] = R[7];
            r[REC_MUX] = mu.x;
            r[REC_MUY] = mu.y;
            r[REC_MUZ] = mu.z;
            r[REC_SX] = sx;
            r[REC_SY] = sy;
            r[REC_OP] = op;
            r[REC_GX] = gx;
            r[REC_GY] = gy;
            // |u| > ru implies alpha < 1/255 (margin 1e-6 relative, exact decision kept
            // for everything inside); disabled when ln(255 o) is tiny.
            const bool safe = log(op / kAlphaMin) >= 1e-3;
            r[REC_ULIM] = safe ? ru * (1.0 + 1e-6) * sx : INFINITY;
            r[REC_VLIM] = safe ? rv * (1.0 + 1e-6) * sy : INFINITY;
            r[REC_RSX] = 1.0 / sx;
            r[REC_RSY] = 1.0 / sy;
            r[REC_OM] = sigmoid(-g[9 * n + i]);  // 1 - o without cancellation
            r[REC_PAD] = 0.0;
            double2* dst = reinterpret_cast<double2*>(a.rec + i * REC_FIELDS);
#pragma unroll
            for (int q = 0; q < REC_FIELDS / 2; ++q) dst[q] = make_double2(r[2 * q], r[2 * q + 1]);
            // fp32 prefilter record: n|num, v1|b1, v2|b2, ulim|vlim (rounded up).
            const double b1 = mx * R[0] + my * R[3] + mz * R[6];
            const double b2 = mx * R[1] + my * R[4] + mz * R[7];
            float4* f = a.recf + i * 4;
            f[0] = make_float4(float(nx_), float(ny_), float(nz_), float(r[REC_NUM]));
            f[1] = make_float4(float(R[0]), float(R[3]), float(R[6]), float(b1));
            f[2] = make_float4(float(R[1]), float(R[4]), float(R[7]), float(b2));
            // + the pixel rect (x0 | x1 << 16, y0 | y1 << 16) for the composite's warp-level cull
            f[3] = make_float4(__double2float_ru(r[REC_ULIM]), __double2float_ru(r[REC_VLIM]),
                               __int_as_float(prect.x | (prect.y << 16)), __int_as_float(prect.z | (prect.w << 16)));
        }
    }
    // block-aggregated statistics: warp sums first (one shared atomic per warp and
    // counter instead of one per thread on the same address)
#ifndef NX_PRE_WARP_STATS
#define NX_PRE_WARP_STATS 1
#endif
    if (NX_PRE_WARP_STATS) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            const unsigned m = __ballot_sync(0xffffffffu, cls == c);
            if (lane == 0 && m) atomicAdd(&s_cnt[c], static_cast<unsigned long long>(__popc(m)));
        }
        const unsigned mk = __ballot_sync(0xffffffffu, kept != 0);
        if (lane == 0 && mk) atomicAdd(&s_cnt[5], static_cast<unsigned long long>(__popc(mk)));
        // rect_tiles <= 2^31 per primitive; a warp's sum fits 64 bits
        unsigned long long rk = static_cast<unsigned long long>(ref_keys), wk2 = static_cast<unsigned long long>(work_keys);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rk += __shfl_down_sync(0xffffffffu, rk, o);
            wk2 += __shfl_down_sync(0xffffffffu, wk2, o);
        }
        if (lane == 0 && rk) atomicAdd(&s_cnt[6], rk);
        if (lane == 0 && wk2) atomicAdd(&s_cnt[7], wk2);
    } else {
        if (cls >= 0) atomicAdd(&s_cnt[cls], 1ull);
        if (kept) atomicAdd(&s_cnt[5], 1ull);
        if (ref_keys) atomicAdd(&s_cnt[6], static_cast<unsigned long long>(ref_keys));
        if (work_keys) atomicAdd(&s_cnt[7], static_cast<unsigned long long>(work_keys));
    }
    __syncthreads();
    if (threadIdx.x < 8 && s_cnt[threadIdx.x]) {
        unsigned long long* dst = threadIdx.x < 5 ? &a.stats->cls[threadIdx.x]
                                  : threadIdx.x == 5 ? &a.stats->straddlers_kept
                                  : threadIdx.x == 6 ? &a.stats->tile_keys
                                                     : &a.stats->work_keys;
        atomicAdd(dst, s_cnt[threadIdx.x]);
    }
}

__global__ void compact_kernel(const int32_t* flag, const int32_t* pos, const uint64_t* key, int64_t n,
                               uint64_t* keys_out, uint32_t* ids_out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) {
        keys_out[pos[i]] = key[i];
        ids_out[pos[i]] = static_cast<uint32_t>(i);
    }
}

// counts over the capacity n: entries past the device count are zero, so a scan over
// the whole capacity yields the right offsets and total.
__device__ __forceinline__ double key_depth(uint64_t k) {  // inverse of depth_key
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

__global__ void rect_counts_kernel(const uint32_t* ids, int64_t n, const int32_t* n_dev, const int4* rect,
                                   int32_t* counts, const uint64_t* keys, FrameStatsD* stats) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t m = n_dev ? min(n, static_cast<int64_t>(*n_dev)) : n;
    if (r < n) counts[r] = r < m ? rect_tiles(rect[ids[r]]) : 0;
    if (keys && r + 1 < m && keys[r] != keys[r + 1]) {  // near-threshold: (depth, id) order of neighbours
        const double d0 = key_depth(keys[r]), d1 = key_depth(keys[r + 1]);
        if (fabs(d1 - d0) <= kNearDepth * fabs(d0)) atomicAdd(&stats->near[NEAR_DEPTH], 1ull);
    }
}

// Conservative cull of a (tile, primitive) key (work lists only): the plane offsets of
// the tile's pixel rays are a projective image of the pixel rectangle, so they lie in the
// quadrilateral of its corner rays' offsets (all four crossing the plane on one side);
// if that quadrilateral, enlarged by the fp32 prefilter's slack, misses the support box
// [-ulim, ulim] x [-vlim, vlim], no pixel of the tile can hit the primitive.
__device__ __forceinline__ bool tile_misses(const float4* f, const EmitCull& cu, int tile) {
    const int tx = tile % cu.tiles_x, ty = tile / cu.tiles_x;
    const int x0 = tx * cu.tile, y0 = ty * cu.tile;
    const int x1 = min(x0 + cu.tile - 1, cu.W - 1), y1 = min(y0 + cu.tile - 1, cu.H - 1);
    const float4 f0 = f[0], f1 = f[1], f2 = f[2], f3 = f[3];
    float umin = 3e38f, umax = -3e38f, vmin = 3e38f, vmax = -3e38f, su = 0.f, sv = 0.f, sgn = 0.f;
    bool valid = true;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float px = ((c & 1) ? x1 : x0) + 0.5f, py = ((c & 2) ? y1 : y0) + 0.5f;
        // pixel_ray (camera.hpp:32-35) in fp32: R^T normalize(((px - cx)/fx, (py - cy)/fy, 1))
        const float a0 = (px - cu.cx) * cu.ifx, a1 = (py - cu.cy) * cu.ify;
        const float rn = rsqrtf(a0 * a0 + a1 * a1 + 1.f);
        const float n0 = a0 * rn, n1 = a1 * rn, n2 = rn;
        const float dx = cu.R[0] * n0 + cu.R[3] * n1 + cu.R[6] * n2;
        const float dy = cu.R[1] * n0 + cu.R[4] * n1 + cu.R[7] * n2;
        const float dz = cu.R[2] * n0 + cu.R[5] * n1 + cu.R[8] * n2;
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
        // the prefilter's slack (fp32 rounding of t and the offsets), doubled for the
        // fp32 ray direction here
        su = fmaxf(su, 2e-4f * (fabsf(ta1) + fabsf(ta) + fabsf(f1.w)) + 2e-7f);
        sv = fmaxf(sv, 2e-4f * (fabsf(ta2) + fabsf(ta) + fabsf(f2.w)) + 2e-7f);
    }
    return valid && (umin > f3.x + su || umax < -f3.x - su || vmin > f3.y + sv || vmax < -f3.y - sv);
}

// One thread per emitted key. Each CTA takes a contiguous range of keys; the owner of
// its first key comes from a 256-ary search of the offsets (one load per thread per
// round, three rounds at 180K primitives); after that, per 256 keys, the primitives that
// start inside the window mark their first key and a block max-scan hands every key its
// owner (the last r with offsets[r] <= k, so zero-count primitives are skipped as in a
// binary search). Counts on the device; keys past the capacity are dropped (the frame is
// re-rendered with a larger capacity before it is read, nx_api.cu frame_settle). Keys
// the cull proves empty go to the sentinel tile n_tiles (sorted past every list).
constexpr int kEmitThreads = 256;
__global__ void __launch_bounds__(kEmitThreads) emit_kernel(const uint32_t* ids, const int32_t* offsets,
                                                            int64_t sorted_cap, const int32_t* n_sorted_dev,
                                                            int64_t key_cap, const int32_t* n_keys_dev,
                                                            const int4* rect, int tiles_x, uint32_t* tile_keys,
                                                            uint32_t* vals, int32_t* tile_counts, const EmitCull cu) {
    __shared__ int32_t s_own[kEmitThreads];
    __shared__ int32_t s_wmax[kEmitThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t n_sorted = min(sorted_cap, static_cast<int64_t>(max(*n_sorted_dev, 0)));
    const int64_t n_keys = n_sorted > 0 ? min(key_cap, static_cast<int64_t>(max(*n_keys_dev, 0))) : 0;
    const int64_t per = ((n_keys + gridDim.x - 1) / gridDim.x + kEmitThreads - 1) / kEmitThreads * kEmitThreads;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * per, k1 = min(n_keys, k0 + per);
    if (k0 >= k1) return;
    // owner of k0 (offsets[0] = 0 <= k0 keeps the invariant offsets[lo] <= k0)
    int64_t lo = 0, hi = n_sorted - 1;
    while (lo < hi) {
        const int64_t step = (hi - lo + kEmitThreads) / kEmitThreads;
        const int64_t r = lo + tid * step;
        const int c = __syncthreads_count(r <= hi && offsets[r] <= k0);
        lo += (c - 1) * step;
        hi = min(hi, lo + step - 1);
    }
    int32_t own = static_cast<int32_t>(lo);
    for (int64_t base = k0; base < k1; base += kEmitThreads) {
        s_own[tid] = -1;
        __syncthreads();
        for (int64_t r0 = own + 1;; r0 += kEmitThreads) {
            const int64_t r = r0 + tid;
            bool more = false;
            if (r < n_sorted) {
                const int64_t o = offsets[r];
                if (o < base + kEmitThreads) {
                    more = true;
                    if (o >= base) atomicMax(&s_own[o - base], static_cast<int32_t>(r));
                }
            }
            if (!__syncthreads_or(more)) break;
        }
        int32_t v = s_own[tid];
        if (tid == 0) v = max(v, own);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v = max(v, y);
        }
        if (lane == 31) s_wmax[wid] = v;
        __syncthreads();
        int32_t pre = -1, all = -1;
#pragma unroll
        for (int w = 0; w < kEmitThreads / 32; ++w) {
            const int32_t m = s_wmax[w];
            if (w < wid) pre = max(pre, m);
            all = max(all, m);
        }
        v = max(v, pre);
        const int64_t k = base + tid;
        if (k < k1) {
            const uint32_t id = ids[v];
            const int4 rc = rect[id];
            const int j = static_cast<int>(k - offsets[v]);
            const int w = rc.y - rc.x + 1;
            int tile = (rc.z + j / w) * tiles_x + rc.x + j % w;
            if (cu.recf && tile_misses(cu.recf + static_cast<int64_t>(id) * 4, cu, tile)) tile = cu.n_tiles;
            tile_keys[k] = static_cast<uint32_t>(tile);
            vals[k] = id;
            if (tile < cu.n_tiles) atomicAdd(&tile_counts[tile], 1);
        }
        own = all;  // the owner of the window's last key
        __syncthreads();
    }
}

// activate()'s checks (primitive.cpp:47-63) over every primitive of a device scene,
// in the reference's order within a primitive; the first failing primitive wins:
// *first = min(id * 8 + what) (what: the index of the failed check).
__global__ void validate_kernel(const double* __restrict__ geom, const float* __restrict__ sh, int64_t n,
                                int64_t nn, unsigned long long* first) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double g[kGeomFields];
#pragma unroll
        for (int k = 0; k < kGeomFields; ++k) g[k] = geom[k * nn + i];
        int what = -1;
        for (int k = 0; k < 3 && what < 0; ++k)
            if (!isfinite(g[k])) what = 0;
        for (int k = 0; k < 4 && what < 0; ++k)
            if (!isfinite(g[3 + k])) what = 1;
        for (int k = 0; k < 2 && what < 0; ++k) {
            if (!isfinite(g[7 + k])) what = 2;
            else if (!isfinite(g[10 + k])) what = 3;
        }
        if (what < 0 && !isfinite(g[9])) what = 4;
        const float* c = sh + i * NX_SH_VALUES;
        for (int k = 0; k < NX_SH_VALUES && what < 0; ++k)
            if (!isfinite(c[k])) what = 5;
        if (what < 0 && !(sqrt(g[3] * g[3] + g[4] * g[4] + g[5] * g[5] + g[6] * g[6]) > 1e-12)) what = 6;
        if (what >= 0) atomicMin(first, (static_cast<unsigned long long>(i) << 3) | static_cast<unsigned>(what));
    }
}

}  // namespace

void launch_validate(const double* geom, const float* sh, int64_t n, unsigned long long* first, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
    validate_kernel<<<blocks, 256, 0, s>>>(geom, sh, n, std::max<int64_t>(n, 1), first);
}

void launch_preprocess(const PreprocessArgs& a, cudaStream_t s) {
    if (a.scene.n <= 0) return;
    const unsigned blocks = static_cast<unsigned>((a.scene.n + kPreThreads - 1) / kPreThreads);
    count_launch();
    preprocess_kernel<<<blocks, kPreThreads, 0, s>>>(a);
}

void launch_compact(const int32_t* flag, const int32_t* pos, const uint64_t* key, int64_t n,
                    uint64_t* keys_out, uint32_t* ids_out, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    compact_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(flag, pos, key, n, keys_out, ids_out);
}

void launch_rect_counts(const uint32_t* ids, int64_t n, const int32_t* n_dev, const int4* rect, int32_t* counts,
                        const uint64_t* sorted_keys, FrameStatsD* stats, cudaStream_t s) {
    if (n <= 0) return;
    count_launch();
    rect_counts_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(ids, n, n_dev, rect, counts,
                                                                               sorted_keys, stats);
}

void launch_emit(const uint32_t* ids, const int32_t* offsets, int64_t sorted_cap, const int32_t* n_sorted_dev,
                 int64_t key_cap, const int32_t* n_keys_dev, const int4* rect, int tiles_x, uint32_t* tile_keys,
                 uint32_t* vals, int32_t* tile_counts, const EmitCull& cull, cudaStream_t s) {
    if (key_cap <= 0 || sorted_cap <= 0) return;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>((key_cap + 255) / 256, static_cast<int64_t>(sms) * 8);
    count_launch();
    emit_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(ids, offsets, sorted_cap, n_sorted_dev, key_cap,
                                                             n_keys_dev, rect, tiles_x, tile_keys, vals, tile_counts,
                                                             cull);
}

}  // namespace nx
