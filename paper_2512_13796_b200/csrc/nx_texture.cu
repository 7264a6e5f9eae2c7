// K7 texture: neural-texture queries at the buffered crossings and the Eq. 7
// composite (texturing_pass, renderer.cpp:207-237).
//
// One thread per top-K slot (pixel-major, slot-minor like build_queries,
// renderer.cpp:177-203); empty slots (id < 0) produce no query. Per query:
//   x = o + t d (fp64, build_queries renderer.cpp:196-198);
//   16-level hash-grid lookup (grid_lookup, hash_grid.cpp:26-83): lattice
//     position, floor and hashing in fp64/int64 exactly as the reference, so
//     the same table rows are gathered; trilinear weights, level fade
//     (downweight, hash_grid.hpp:28-31) and accumulation in fp32;
//   bias-free ReLU MLP 32->64->64->48 in fp32 from shared-memory weights
//     (TextureMlp::forward, mlp.cpp:24-43);
//   degree-3 SH colour with the ray direction (eval_sh, sh.hpp:46-57).
// The CTA then forms final = base + sum_j W[p,j] * texture[p,j] for its pixels
// (renderer.cpp:219-236) from the slot colours it holds in shared memory.
#include <cstdlib>
#include <cstring>

#include "nx_composite.cuh"

namespace nx {

namespace {

constexpr int kTexThreads = 128;

__device__ __forceinline__ uint32_t map_positive32(long long x) {  // hash_grid.hpp:12-14
    return x > 0 ? static_cast<uint32_t>(2 * x - 1) : static_cast<uint32_t>(-2 * x);
}
__device__ __forceinline__ uint32_t hash_cell(long long ix, long long iy, long long iz, uint32_t mask) {
    // hash_grid.hpp:17-23, 32-bit wrapping
    return (map_positive32(ix) ^ (map_positive32(iy) * 2654435761u) ^ (map_positive32(iz) * 805459861u)) & mask;
}

__device__ __forceinline__ void sh_basis_f(const double* d, float* b) {  // sh.hpp:11-40
    const float x = static_cast<float>(d[0]), y = static_cast<float>(d[1]), z = static_cast<float>(d[2]);
    const float xx = x * x, yy = y * y, zz = z * z;
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
}

// NIN / NH / F: compile-time fast path (32, 64, 2) or 0 = runtime (generic shapes).
template <int NIN, int NH, int F>
__global__ void __launch_bounds__(kTexThreads) texture_kernel(const TextureArgs a) {
    constexpr int kMaxIn = NIN ? NIN : 64;
    constexpr int kMaxH = NH ? NH : 128;
    extern __shared__ float smem[];
    const nx_field_desc& fd = a.scene.field;
    const int nin = NIN ? NIN : fd.levels * fd.features;
    const int nh = NH ? NH : fd.n_hidden;
    const int nf = F ? F : fd.features;
    float* sW1 = smem;
    float* sW2 = sW1 + nh * nin;
    float* sW3 = sW2 + nh * nh;
    float* s_tex = sW3 + NX_SH_VALUES * nh;  // blockDim * 3
    for (int e = threadIdx.x; e < nh * nin; e += blockDim.x) sW1[e] = a.scene.w1[e];
    for (int e = threadIdx.x; e < nh * nh; e += blockDim.x) sW2[e] = a.scene.w2[e];
    for (int e = threadIdx.x; e < NX_SH_VALUES * nh; e += blockDim.x) sW3[e] = a.scene.w3[e];
    __syncthreads();

    const int K = a.fb.K;
    const int W = a.cam.W;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
    const int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    float rgb[3] = {0.f, 0.f, 0.f};
    bool valid = false;
    if (slot < total && a.fb.ids[slot] >= 0) {
        valid = true;
        const int64_t pix = slot / K;
        const int px = static_cast<int>(pix % W), py = static_cast<int>(pix / W);
        double dir[3];
        pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
        const double t = a.fb.depths[slot];
        const double x0 = a.cam.o[0] + t * dir[0];
        const double x1 = a.cam.o[1] + t * dir[1];
        const double x2 = a.cam.o[2] + t * dir[2];
        const uint32_t T = 1u << fd.log2_table;
        const uint32_t mask = T - 1u;
        const double f = a.cam.fx;
        float feats[kMaxIn];
        double s = fd.base_scale;
#pragma unroll
        for (int l = 0; l < (NIN ? NIN / (F ? F : 1) : 64); ++l) {
            if (!NIN && l >= fd.levels) break;
            const double p0 = s * x0, p1 = s * x1, p2 = s * x2;
            const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
            const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                            b2 = static_cast<long long>(fl2);
            const float fr0 = static_cast<float>(p0 - fl0), fr1 = static_cast<float>(p1 - fl1),
                        fr2 = static_cast<float>(p2 - fl2);
            float dw = 1.0f;
            if (!a.st.no_downweight) {
                const double r = f / (s * t);
                dw = 1.0f - __expf(static_cast<float>(-r * r / (2.0 * M_PI)));
            }
            const float wx[2] = {1.0f - fr0, fr0}, wy[2] = {1.0f - fr1, fr1}, wz[2] = {1.0f - fr2, fr2};
            const size_t slab = static_cast<size_t>(l) * T;
            if (F == 2) {
                const float2* tab = reinterpret_cast<const float2*>(a.scene.table);
                float g0 = 0.f, g1 = 0.f;
#pragma unroll
                for (int ci = 0; ci < 8; ++ci) {
                    const uint32_t row = hash_cell(b0 + (ci & 1), b1 + ((ci >> 1) & 1), b2 + ((ci >> 2) & 1), mask);
                    const float w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
                    const float2 v = __ldg(tab + slab + row);
                    g0 += w * v.x;
                    g1 += w * v.y;
                }
                feats[2 * l] = g0 * dw;
                feats[2 * l + 1] = g1 * dw;
            } else {
                for (int fi = 0; fi < nf; ++fi) feats[l * nf + fi] = 0.f;
                for (int ci = 0; ci < 8; ++ci) {
                    const uint32_t row = hash_cell(b0 + (ci & 1), b1 + ((ci >> 1) & 1), b2 + ((ci >> 2) & 1), mask);
                    const float w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
                    for (int fi = 0; fi < nf; ++fi)
                        feats[l * nf + fi] += w * __ldg(a.scene.table + (slab + row) * nf + fi);
                }
                for (int fi = 0; fi < nf; ++fi) feats[l * nf + fi] *= dw;
            }
            s *= fd.growth;
        }
        // MLP (mlp.cpp:24-43)
        float h1[kMaxH];
#pragma unroll
        for (int o = 0; o < kMaxH; ++o) {
            if (!NH && o >= nh) break;
            float acc = 0.f;
            const float* row = sW1 + o * nin;
#pragma unroll
            for (int i = 0; i < kMaxIn; ++i) {
                if (!NIN && i >= nin) break;
                acc = fmaf(row[i], feats[i], acc);
            }
            h1[o] = fmaxf(acc, 0.f);
        }
        float h2[kMaxH];
#pragma unroll
        for (int o = 0; o < kMaxH; ++o) {
            if (!NH && o >= nh) break;
            float acc = 0.f;
            const float* row = sW2 + o * nh;
#pragma unroll
            for (int i = 0; i < kMaxH; ++i) {
                if (!NH && i >= nh) break;
                acc = fmaf(row[i], h1[i], acc);
            }
            h2[o] = fmaxf(acc, 0.f);
        }
        float b[16];
        sh_basis_f(dir, b);
        float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            float y[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float acc = 0.f;
                const float* row = sW3 + (k * 3 + c) * nh;
#pragma unroll
                for (int i = 0; i < kMaxH; ++i) {
                    if (!NH && i >= nh) break;
                    acc = fmaf(row[i], h2[i], acc);
                }
                y[c] = acc;
            }
            c0 = fmaf(y[0], b[k], c0);
            c1 = fmaf(y[1], b[k], c1);
            c2 = fmaf(y[2], b[k], c2);
        }
        rgb[0] = fmaxf(0.5f + c0, 0.f);
        rgb[1] = fmaxf(0.5f + c1, 0.f);
        rgb[2] = fmaxf(0.5f + c2, 0.f);
    }
    if (slot < total) {
        a.fb.texture[slot * 3 + 0] = rgb[0];
        a.fb.texture[slot * 3 + 1] = rgb[1];
        a.fb.texture[slot * 3 + 2] = rgb[2];
    }
    s_tex[threadIdx.x * 3 + 0] = rgb[0];
    s_tex[threadIdx.x * 3 + 1] = rgb[1];
    s_tex[threadIdx.x * 3 + 2] = rgb[2];
    const int nq = __syncthreads_count(valid);
    if (threadIdx.x == 0 && nq) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(nq));
    // Eq. 7 composite for the pixels whose slots this block holds.
    const int ppb = blockDim.x / K;
    if (threadIdx.x < ppb) {
        const int64_t pix = static_cast<int64_t>(blockIdx.x) * ppb + threadIdx.x;
        if (pix < static_cast<int64_t>(a.cam.W) * a.cam.H) {
            double acc0 = a.fb.base[pix * 3 + 0], acc1 = a.fb.base[pix * 3 + 1], acc2 = a.fb.base[pix * 3 + 2];
            for (int j = 0; j < K; ++j) {
                const int64_t sl = pix * K + j;
                if (a.fb.ids[sl] < 0) continue;
                const double w = a.fb.weights[sl];
                const float* tc = s_tex + (threadIdx.x * K + j) * 3;
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

__global__ void copy_base_kernel(const float* base, float* final_img, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) final_img[i] = base[i];
}

template <int NIN, int NH, int F>
void launch_tex(const TextureArgs& a, cudaStream_t s) {
    const int K = a.fb.K;
    const int threads = (kTexThreads / K) * K;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
    const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
    const int nin = a.scene.field.levels * a.scene.field.features, nh = a.scene.field.n_hidden;
    const size_t smem = sizeof(float) * (static_cast<size_t>(nh) * nin + nh * nh + NX_SH_VALUES * nh + threads * 3);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(texture_kernel<NIN, NH, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    count_launch();
    texture_kernel<NIN, NH, F><<<blocks, threads, smem, s>>>(a);
}


// ---------------------------------------------------------------- NX_PRECISION_F64
// texturing_pass (renderer.cpp:207-237) at the reference's precision: one thread per
// pixel; per buffered slot the query of build_queries (renderer.cpp:177-203), grid_lookup
// (hash_grid.cpp:26-83) on the fp64 table, TextureMlp::forward (mlp.cpp:24-43) on the
// fp64 weights, eval_sh (sh.hpp:46-57) in fp64, then Eq. 7 on the fp64 base. The
// reference's operation order throughout (its decoder sums are reassociated by its
// compiler flags, so the last bits may differ: ~1e-16 relative).
constexpr int kF64MaxIn = 64, kF64MaxHidden = 128;

__device__ __forceinline__ uint32_t f64_map_positive(long long x) {  // hash_grid.hpp:12-14
    return x > 0 ? static_cast<uint32_t>(2 * x - 1) : static_cast<uint32_t>(-2 * x);
}

__global__ void __launch_bounds__(64) texture_f64_kernel(const TextureArgs a) {
    const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H;
    const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pix >= npix) return;
    const int K = a.fb.K;
    const nx_field_desc& fd = a.scene.field;
    const int L = fd.levels, F = fd.features, nin = L * F, nh = fd.n_hidden;
    const uint32_t T = 1u << fd.log2_table, mask = T - 1u;
    const int px = static_cast<int>(pix % a.cam.W), py = static_cast<int>(pix / a.cam.W);
    double dir[3];
    pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
    double acc[3] = {a.fb.base64[pix * 3 + 0], a.fb.base64[pix * 3 + 1], a.fb.base64[pix * 3 + 2]};
    int n_q = 0;
    for (int j = 0; j < K; ++j) {
        const int64_t sl = pix * K + j;
        if (a.fb.ids[sl] < 0) {
            for (int c = 0; c < 3; ++c) {
                a.fb.texture64[sl * 3 + c] = 0.0;
                a.fb.texture[sl * 3 + c] = 0.f;
            }
            continue;
        }
        ++n_q;
        const double t = a.fb.depths[sl];
        const double x[3] = {a.cam.o[0] + t * dir[0], a.cam.o[1] + t * dir[1], a.cam.o[2] + t * dir[2]};
        const double f = a.cam.fx;
        double feats[kF64MaxIn];
        double s = fd.base_scale;
        for (int l = 0; l < L; ++l, s *= fd.growth) {
            const double p0 = s * x[0], p1 = s * x[1], p2 = s * x[2];
            const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
            const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                            b2 = static_cast<long long>(fl2);
            const double fr[3] = {p0 - fl0, p1 - fl1, p2 - fl2};
            double dw = 1.0;
            if (!a.st.no_downweight) {  // downweight (hash_grid.hpp:28-31)
                const double r = f / (s * t);
                dw = 1.0 - exp(-r * r / (2.0 * M_PI));
            }
            const double wx[2] = {1.0 - fr[0], fr[0]}, wy[2] = {1.0 - fr[1], fr[1]}, wz[2] = {1.0 - fr[2], fr[2]};
            for (int fi = 0; fi < F; ++fi) feats[l * F + fi] = 0.0;
            const size_t slab = static_cast<size_t>(l) * T;
            for (int ci = 0; ci < 8; ++ci) {
                const uint32_t row = (f64_map_positive(b0 + (ci & 1)) ^
                                      (f64_map_positive(b1 + ((ci >> 1) & 1)) * 2654435761u) ^
                                      (f64_map_positive(b2 + ((ci >> 2) & 1)) * 805459861u)) & mask;
                const double w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
                const double* feat = a.scene.table64 + (slab + row) * F;
                for (int fi = 0; fi < F; ++fi) feats[l * F + fi] += w * __ldg(feat + fi);
            }
            for (int fi = 0; fi < F; ++fi) feats[l * F + fi] *= dw;
        }
        double h1[kF64MaxHidden], h2[kF64MaxHidden], y[NX_SH_VALUES];
        for (int o = 0; o < nh; ++o) {
            double v = 0.0;
            for (int i = 0; i < nin; ++i) v += __ldg(a.scene.w1_64 + o * nin + i) * feats[i];
            h1[o] = v > 0.0 ? v : 0.0;
        }
        for (int o = 0; o < nh; ++o) {
            double v = 0.0;
            for (int i = 0; i < nh; ++i) v += __ldg(a.scene.w2_64 + o * nh + i) * h1[i];
            h2[o] = v > 0.0 ? v : 0.0;
        }
        for (int o = 0; o < NX_SH_VALUES; ++o) {
            double v = 0.0;
            for (int i = 0; i < nh; ++i) v += __ldg(a.scene.w3_64 + o * nh + i) * h2[i];
            y[o] = v;
        }
        double rgb[3];
        eval_sh_f64(y, dir, 3, rgb);  // field_forward: always degree 3 (texture_field.cpp:33)
        const double w = a.fb.weights[sl];
        for (int c = 0; c < 3; ++c) {
            a.fb.texture64[sl * 3 + c] = rgb[c];
            a.fb.texture[sl * 3 + c] = static_cast<float>(rgb[c]);
            acc[c] += w * rgb[c];
        }
    }
    for (int c = 0; c < 3; ++c) {
        a.fb.final64[pix * 3 + c] = acc[c];
        a.fb.final_img[pix * 3 + c] = static_cast<float>(acc[c]);
    }
    if (n_q) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_q));
}


// The reference field shape (16 levels x 2 features -> 64 -> 64 -> 48) at NX_PRECISION_F64:
// one thread per slot, the fp64 weights in shared memory (broadcast reads), features in
// registers, layers 1 and 2 interleaved — h1[o1] is formed and immediately folded into the
// h2 accumulators, so every h2[o2] still sums its 64 terms in ascending order like
// TextureMlp::forward (mlp.cpp:24-43) — in two halves of h2 to bound the registers (layer 1
// is formed twice). Then eval_sh in fp64; Eq. 7 runs per pixel in final_f64_kernel.
constexpr int kF64In = 32, kF64Hid = 64, kF64Half = 32;
constexpr int kF64WBytes = (kF64Hid * kF64In + kF64Hid * kF64Hid + NX_SH_VALUES * kF64Hid) * 8;  // 72 KB

__global__ void __launch_bounds__(128) texture_f64_slot_kernel(const TextureArgs a) {
    extern __shared__ __align__(16) double wsm[];
    double* w1 = wsm;
    double* w2 = w1 + kF64Hid * kF64In;
    double* w3 = w2 + kF64Hid * kF64Hid;
    for (int i = threadIdx.x; i < kF64Hid * kF64In; i += blockDim.x) w1[i] = a.scene.w1_64[i];
    for (int i = threadIdx.x; i < kF64Hid * kF64Hid; i += blockDim.x) w2[i] = a.scene.w2_64[i];
    for (int i = threadIdx.x; i < NX_SH_VALUES * kF64Hid; i += blockDim.x) w3[i] = a.scene.w3_64[i];
    __syncthreads();
    const int K = a.fb.K;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (sl >= total) return;
    if (a.fb.ids[sl] < 0) {
        for (int c = 0; c < 3; ++c) {
            a.fb.texture64[sl * 3 + c] = 0.0;
            a.fb.texture[sl * 3 + c] = 0.f;
        }
        return;
    }
    const nx_field_desc& fd = a.scene.field;
    const uint32_t T = 1u << fd.log2_table, mask = T - 1u;
    const int64_t pix = sl / K;
    const int px = static_cast<int>(pix % a.cam.W), py = static_cast<int>(pix / a.cam.W);
    double dir[3];
    pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
    const double t = a.fb.depths[sl];
    const double x[3] = {a.cam.o[0] + t * dir[0], a.cam.o[1] + t * dir[1], a.cam.o[2] + t * dir[2]};
    const double f = a.cam.fx;
    double feats[kF64In];
    double s = fd.base_scale;
#pragma unroll
    for (int l = 0; l < kF64In / 2; ++l, s *= fd.growth) {  // grid_lookup (hash_grid.cpp:26-83), F == 2
        const double p0 = s * x[0], p1 = s * x[1], p2 = s * x[2];
        const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
        const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                        b2 = static_cast<long long>(fl2);
        const double fr0 = p0 - fl0, fr1 = p1 - fl1, fr2 = p2 - fl2;
        double dw = 1.0;
        if (!a.st.no_downweight) {  // downweight (hash_grid.hpp:28-31)
            const double r = f / (s * t);
            dw = 1.0 - exp(-r * r / (2.0 * M_PI));
        }
        const double wx[2] = {1.0 - fr0, fr0}, wy[2] = {1.0 - fr1, fr1}, wz[2] = {1.0 - fr2, fr2};
        double a0 = 0.0, a1 = 0.0;
        const double2* slab = reinterpret_cast<const double2*>(a.scene.table64) + static_cast<size_t>(l) * T;
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
            const uint32_t row = (f64_map_positive(b0 + (ci & 1)) ^ (f64_map_positive(b1 + ((ci >> 1) & 1)) * 2654435761u) ^
                                  (f64_map_positive(b2 + ((ci >> 2) & 1)) * 805459861u)) & mask;
            const double w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
            const double2 v = __ldg(slab + row);
            a0 += w * v.x;
            a1 += w * v.y;
        }
        feats[2 * l] = a0 * dw;
        feats[2 * l + 1] = a1 * dw;
    }
    double h2[kF64Hid];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        double acc2[kF64Half];
#pragma unroll
        for (int o2 = 0; o2 < kF64Half; ++o2) acc2[o2] = 0.0;
#pragma unroll 1
        for (int o1 = 0; o1 < kF64Hid; ++o1) {
            double h = 0.0;
#pragma unroll
            for (int i = 0; i < kF64In; ++i) h += w1[o1 * kF64In + i] * feats[i];
            h = h > 0.0 ? h : 0.0;
#pragma unroll
            for (int o2 = 0; o2 < kF64Half; ++o2) acc2[o2] += w2[(half * kF64Half + o2) * kF64Hid + o1] * h;
        }
#pragma unroll
        for (int o2 = 0; o2 < kF64Half; ++o2) h2[half * kF64Half + o2] = acc2[o2] > 0.0 ? acc2[o2] : 0.0;
    }
    double y[NX_SH_VALUES];
#pragma unroll 4
    for (int o = 0; o < NX_SH_VALUES; ++o) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < kF64Hid; ++i) v += w3[o * kF64Hid + i] * h2[i];
        y[o] = v;
    }
    double rgb[3];
    eval_sh_f64(y, dir, 3, rgb);  // field_forward: always degree 3 (texture_field.cpp:33)
    for (int c = 0; c < 3; ++c) {
        a.fb.texture64[sl * 3 + c] = rgb[c];
        a.fb.texture[sl * 3 + c] = static_cast<float>(rgb[c]);
    }
}

// Eq. 7 per pixel (renderer.cpp:219-236): final = base + sum_j W[p,j] texture[p,j], slot order.
__global__ void final_f64_kernel(const TextureArgs a) {
    const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H;
    const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pix >= npix) return;
    const int K = a.fb.K;
    double acc[3] = {a.fb.base64[pix * 3 + 0], a.fb.base64[pix * 3 + 1], a.fb.base64[pix * 3 + 2]};
    int n_q = 0;
    for (int j = 0; j < K; ++j) {
        const int64_t sl = pix * K + j;
        if (a.fb.ids[sl] < 0) continue;
        ++n_q;
        const double w = a.fb.weights[sl];
        for (int c = 0; c < 3; ++c) acc[c] += w * a.fb.texture64[sl * 3 + c];
    }
    for (int c = 0; c < 3; ++c) {
        a.fb.final64[pix * 3 + c] = acc[c];
        a.fb.final_img[pix * 3 + c] = static_cast<float>(acc[c]);
    }
    if (n_q) atomicAdd(&a.stats->queries, static_cast<unsigned long long>(n_q));
}

__global__ void copy_base64_kernel(const double* base64, const float* base, double* final64, float* final_img,
                                   int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        final64[i] = base64[i];
        final_img[i] = base[i];
    }
}

}  // namespace

int launch_texture(const TextureArgs& a, cudaStream_t s) {
    const int64_t npix = static_cast<int64_t>(a.cam.W) * a.cam.H;
    if (a.fb.final64 && a.scene.table64) {  // NX_PRECISION_F64 render
        if (npix == 0) return NX_OK;
        const nx_field_desc& fd = a.scene.field;
        if (fd.levels * fd.features > kF64MaxIn || fd.n_hidden > kF64MaxHidden) return NX_UNSUPPORTED;
        count_launch();
        if (a.fb.K == 0) {
            copy_base64_kernel<<<static_cast<unsigned>((npix * 3 + 255) / 256), 256, 0, s>>>(
                a.fb.base64, a.fb.base, a.fb.final64, a.fb.final_img, npix * 3);
        } else if (fd.levels == kF64In / 2 && fd.features == 2 && fd.n_hidden == kF64Hid) {
            const int64_t total = npix * a.fb.K;
            cudaFuncSetAttribute(texture_f64_slot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kF64WBytes);
            count_launch();
            texture_f64_slot_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, kF64WBytes, s>>>(a);
            final_f64_kernel<<<static_cast<unsigned>((npix + 255) / 256), 256, 0, s>>>(a);
        } else {
            texture_f64_kernel<<<static_cast<unsigned>((npix + 63) / 64), 64, 0, s>>>(a);
        }
        return NX_OK;
    }
    if (a.fb.K == 0) {
        if (npix * 3 > 0)
            count_launch(), copy_base_kernel<<<static_cast<unsigned>((npix * 3 + 255) / 256), 256, 0, s>>>(a.fb.base, a.fb.final_img,
                                                                                         npix * 3);
        return NX_OK;
    }
    const nx_field_desc& fd = a.scene.field;
    const int nin = fd.levels * fd.features;
    // NX_TEXTURE_PATH=simt forces the SIMT MLP (validation of the tensor-core path).
    static const bool force_simt = [] {
        const char* e = getenv("NX_TEXTURE_PATH");
        return e && strcmp(e, "simt") == 0;
    }();
    if (!force_simt && texture_tc_supported(fd)) return launch_texture_tc(a, s);
    if (nin == 32 && fd.features == 2 && fd.n_hidden == 64) {
        launch_tex<32, 64, 2>(a, s);
        return NX_OK;
    }
    if (nin > 64 || fd.n_hidden > 128 || fd.levels > 64) return NX_UNSUPPORTED;
    launch_tex<0, 0, 0>(a, s);
    return NX_OK;
}

}  // namespace nx
