// Field branch of render_backward (renderer.cpp:261-284): for every buffered slot,
// the colour gradient dL/drgb = w * dL/dfinal + dL/dtexture, then
// field_backward_batch (texture_field.cpp:77-146): grid_lookup (hash_grid.cpp:
// 26-83) + TextureMlp::forward (mlp.cpp:24-43) recomputed, eval_sh_backward
// (sh.hpp:76-83), TextureMlp::backward (mlp.cpp:45-90) and grid_lookup_backward
// (hash_grid.hpp:85-124). Outputs: table / MLP weight gradients (exact
// order-independent accumulators, nx_xacc.cuh, read back into the fp64 gradients) and, per slot, dL/dt + dot(dL/dx, dir) — the crossing-depth gradient the
// compositing branch folds into intersect_backward (renderer.cpp:283-284).
//
// This file holds the general-shape SIMT variant (one thread per slot, fp64
// throughout like the reference, weights read through L1). It is the validation
// twin of the tensor-core variant (nx_field_backward_tc.cu) and the path for
// field shapes other than 16 levels x 2 features x 64 hidden.
#include <cstdlib>
#include <cstring>

#include "nx_internal.cuh"

namespace nx {

namespace {

constexpr int kMaxIn = 64;
constexpr int kMaxHidden = 128;

__device__ __forceinline__ uint32_t map_positive32(long long x) {  // hash_grid.hpp:12-14
    return x > 0 ? static_cast<uint32_t>(2 * x - 1) : static_cast<uint32_t>(-2 * x);
}
__device__ __forceinline__ uint32_t hash_cell(long long ix, long long iy, long long iz, uint32_t mask) {
    return (map_positive32(ix) ^ (map_positive32(iy) * 2654435761u) ^ (map_positive32(iz) * 805459861u)) & mask;
}

// sh_basis (sh.hpp:11-40), degree 3, fp64.
__device__ __forceinline__ void sh_basis_d(const double* d, double* b) {
    const double x = d[0], y = d[1], z = d[2];
    const double xx = x * x, yy = y * y, zz = z * z;
    b[0] = 0.28209479177387814;
    b[1] = -0.4886025119029199 * y;
    b[2] = 0.4886025119029199 * z;
    b[3] = -0.4886025119029199 * x;
    b[4] = 1.0925484305920792 * x * y;
    b[5] = -1.0925484305920792 * y * z;
    b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    b[7] = -1.0925484305920792 * x * z;
    b[8] = 0.5462742152960396 * (xx - yy);
    b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    b[10] = 2.890611442640554 * x * y * z;
    b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    b[14] = 1.445305721320277 * z * (xx - yy);
    b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
}

__global__ void __launch_bounds__(128) field_bwd_simt_kernel(const FieldBwdArgs a, const Xacc tacc, const Xacc wacc) {
    const nx_field_desc& fd = a.scene.field;
    const int K = a.fb.K;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * K;
    const int64_t sl = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (sl >= total) return;
    if (a.fb.ids[sl] < 0) {
        a.d_t_slot[sl] = 0.0;
        return;
    }
    const int64_t pix = sl / K;
    const int px = static_cast<int>(pix % a.cam.W), py = static_cast<int>(pix / a.cam.W);
    // dL/drgb of the query (renderer.cpp:266-276)
    const double w = a.fb.weights[sl];
    double drgb[3];
    for (int c = 0; c < 3; ++c) {
        double g = 0.0;
        if (a.d_final) g += w * a.d_final[pix * 3 + c];
        if (a.d_texture) g += a.d_texture[sl * 3 + c];
        drgb[c] = g;
    }
    double dir[3];
    pixel_dir(a.cam, px + 0.5, py + 0.5, dir);
    const double t = a.fb.depths[sl];
    const double x[3] = {a.cam.o[0] + t * dir[0], a.cam.o[1] + t * dir[1], a.cam.o[2] + t * dir[2]};  // build_queries
    const double f = a.cam.fx;
    const int L = fd.levels, F = fd.features, nin = L * F, nh = fd.n_hidden;
    const uint32_t T = 1u << fd.log2_table, mask = T - 1u;
    const float* tab = a.scene.table;

    // ---- grid_lookup (hash_grid.cpp:26-83)
    double feats[kMaxIn];
    {
        double s = fd.base_scale;
        for (int l = 0; l < L; ++l, s *= fd.growth) {
            const double p0 = s * x[0], p1 = s * x[1], p2 = s * x[2];
            const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
            const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                            b2 = static_cast<long long>(fl2);
            const double fr[3] = {p0 - fl0, p1 - fl1, p2 - fl2};
            double dw = 1.0;
            if (!a.st.no_downweight) {
                const double r = f / (s * t);
                dw = 1.0 - exp(-r * r / (2.0 * M_PI));
            }
            for (int fi = 0; fi < F; ++fi) feats[l * F + fi] = 0.0;
            const size_t slab = static_cast<size_t>(l) * T;
            for (int ci = 0; ci < 8; ++ci) {
                const uint32_t row = hash_cell(b0 + (ci & 1), b1 + ((ci >> 1) & 1), b2 + ((ci >> 2) & 1), mask);
                const double cw = ((ci & 1) ? fr[0] : 1.0 - fr[0]) * ((ci & 2) ? fr[1] : 1.0 - fr[1]) *
                                  ((ci & 4) ? fr[2] : 1.0 - fr[2]);
                for (int fi = 0; fi < F; ++fi) feats[l * F + fi] += cw * __ldg(tab + (slab + row) * F + fi);
            }
            for (int fi = 0; fi < F; ++fi) feats[l * F + fi] *= dw;
        }
    }
    // ---- TextureMlp::forward (mlp.cpp:24-43)
    double h1[kMaxHidden], h2[kMaxHidden];
    for (int o = 0; o < nh; ++o) {
        double acc = 0.0;
        for (int i = 0; i < nin; ++i) acc += static_cast<double>(__ldg(a.scene.w1 + o * nin + i)) * feats[i];
        h1[o] = acc > 0.0 ? acc : 0.0;
    }
    for (int o = 0; o < nh; ++o) {
        double acc = 0.0;
        for (int i = 0; i < nh; ++i) acc += static_cast<double>(__ldg(a.scene.w2 + o * nh + i)) * h1[i];
        h2[o] = acc > 0.0 ? acc : 0.0;
    }
    double basis[16];
    sh_basis_d(dir, basis);
    // eval_sh_cached (sh.hpp:61-73): clamp mask of 0.5 + sum_k y[k*3+c] basis_k
    double dy[NX_SH_VALUES];
    {
        double accs[3] = {0.5, 0.5, 0.5};
        for (int o = 0; o < NX_SH_VALUES; ++o) {
            double acc = 0.0;
            for (int i = 0; i < nh; ++i) acc += static_cast<double>(__ldg(a.scene.w3 + o * nh + i)) * h2[i];
            accs[o % 3] += acc * basis[o / 3];
        }
        // eval_sh_backward (sh.hpp:76-83)
        for (int o = 0; o < NX_SH_VALUES; ++o) {
            const int c = o % 3;
            dy[o] = accs[c] >= 0.0 ? drgb[c] * basis[o / 3] : 0.0;
        }
    }
    // ---- TextureMlp::backward (mlp.cpp:45-90)
    double dh[kMaxHidden];
    for (int i = 0; i < nh; ++i) dh[i] = 0.0;
    for (int o = 0; o < NX_SH_VALUES; ++o) {
        const double g = dy[o];
        if (g == 0.0) continue;
        for (int i = 0; i < nh; ++i) {
            if (h2[i] != 0.0) xacc_add(wacc, nh * nin + nh * nh + o * nh + i, g * h2[i]);
            dh[i] += g * static_cast<double>(__ldg(a.scene.w3 + o * nh + i));
        }
    }
    for (int i = 0; i < nh; ++i)
        if (h2[i] <= 0.0) dh[i] = 0.0;
    // d_h1 into h2's storage (h2 is no longer needed)
    double* dh1 = h2;
    for (int i = 0; i < nh; ++i) dh1[i] = 0.0;
    for (int o = 0; o < nh; ++o) {
        const double g = dh[o];
        if (g == 0.0) continue;
        for (int i = 0; i < nh; ++i) {
            if (h1[i] != 0.0) xacc_add(wacc, nh * nin + o * nh + i, g * h1[i]);
            dh1[i] += g * static_cast<double>(__ldg(a.scene.w2 + o * nh + i));
        }
    }
    for (int i = 0; i < nh; ++i)
        if (h1[i] <= 0.0) dh1[i] = 0.0;
    double dfeat[kMaxIn];
    for (int i = 0; i < nin; ++i) dfeat[i] = 0.0;
    for (int o = 0; o < nh; ++o) {
        const double g = dh1[o];
        if (g == 0.0) continue;
        for (int i = 0; i < nin; ++i) {
            if (feats[i] != 0.0) xacc_add(wacc, o * nin + i, g * feats[i]);
            dfeat[i] += g * static_cast<double>(__ldg(a.scene.w1 + o * nin + i));
        }
    }
    // ---- grid_lookup_backward (hash_grid.hpp:85-124)
    double dx[3] = {0.0, 0.0, 0.0}, dt = 0.0;
    {
        double s = fd.base_scale;
        for (int l = 0; l < L; ++l, s *= fd.growth) {
            const double p0 = s * x[0], p1 = s * x[1], p2 = s * x[2];
            const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
            const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                            b2 = static_cast<long long>(fl2);
            const double fr[3] = {p0 - fl0, p1 - fl1, p2 - fl2};
            double dw = 1.0;
            if (!a.st.no_downweight) {
                const double r = f / (s * t);
                dw = 1.0 - exp(-r * r / (2.0 * M_PI));
            }
            const double* g = dfeat + l * F;
            const size_t slab = static_cast<size_t>(l) * T;
            double d_dw = 0.0, dp[3] = {0.0, 0.0, 0.0};
            for (int ci = 0; ci < 8; ++ci) {
                const uint32_t row = hash_cell(b0 + (ci & 1), b1 + ((ci >> 1) & 1), b2 + ((ci >> 2) & 1), mask);
                const double wx = (ci & 1) ? fr[0] : 1.0 - fr[0];
                const double wy = (ci & 2) ? fr[1] : 1.0 - fr[1];
                const double wz = (ci & 4) ? fr[2] : 1.0 - fr[2];
                const double cw = wx * wy * wz;
                double gdotf = 0.0;
                for (int fi = 0; fi < F; ++fi) {
                    const double up = g[fi] * dw;
                    if (up * cw != 0.0) xacc_add(tacc, static_cast<int64_t>((slab + row) * F + fi), up * cw);
                    gdotf += g[fi] * static_cast<double>(__ldg(tab + (slab + row) * F + fi));
                }
                const double updotf = gdotf * dw;
                dp[0] += updotf * ((ci & 1) ? 1.0 : -1.0) * wy * wz;
                dp[1] += updotf * wx * ((ci & 2) ? 1.0 : -1.0) * wz;
                dp[2] += updotf * wx * wy * ((ci & 4) ? 1.0 : -1.0);
                d_dw += gdotf * cw;
            }
            dx[0] += s * dp[0];
            dx[1] += s * dp[1];
            dx[2] += s * dp[2];
            if (!a.st.no_downweight) {
                const double r = f / (s * t);
                dt += d_dw * (dw - 1.0) * r * r / (M_PI * t);
            }
        }
    }
    // renderer.cpp:283-284: d_t_total = d_t + dot(d_x, dir)
    a.d_t_slot[sl] = dt + (dx[0] * dir[0] + dx[1] * dir[1] + dx[2] * dir[2]);
}

// g_w1 / g_w2 / g_w3 += the exact weight-gradient sums ([w1 | w2 | w3] in one accumulator).
__global__ void take_weights_kernel(const Xacc acc, int64_t n1, int64_t n2, double* g_w1, double* g_w2, double* g_w3) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= acc.m) return;
    const double v = xacc_take(acc, i);
    if (v == 0.0) return;
    if (i < n1) g_w1[i] += v;
    else if (i < n1 + n2) g_w2[i - n1] += v;
    else g_w3[i - n1 - n2] += v;
}

}  // namespace

int launch_field_backward_simt(const FieldBwdArgs& a, cudaStream_t s) {
    const nx_field_desc& fd = a.scene.field;
    if (fd.levels * fd.features > kMaxIn || fd.n_hidden > kMaxHidden) return NX_UNSUPPORTED;
    const int64_t total = static_cast<int64_t>(a.cam.W) * a.cam.H * a.fb.K;
    if (total == 0) return NX_OK;
    const int64_t nin = static_cast<int64_t>(fd.levels) * fd.features, nh = fd.n_hidden;
    const int64_t n1 = nh * nin, n2 = nh * nh, nw = n1 + n2 + NX_SH_VALUES * nh;
    const int64_t nt = static_cast<int64_t>(fd.levels) * (int64_t(1) << fd.log2_table) * fd.features;
    FieldBwdScratch& sc = *a.scratch;
    if (int st = sc.table_acc(nt, s)) return st;
    if (int st = sc.weight_acc(nw, s)) return st;
    const Xacc tacc{sc.tx, nt}, wacc{sc.wx, nw};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    count_launch(3);
    field_bwd_simt_kernel<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s>>>(a, tacc, wacc);
    take_table_kernel<<<8 * sms, 256, 0, s>>>(a.g_table, tacc);
    take_weights_kernel<<<static_cast<unsigned>((nw + 255) / 256), 256, 0, s>>>(wacc, n1, n2, a.g_w1, a.g_w2, a.g_w3);
    return NX_OK;
}

int launch_field_backward(const FieldBwdArgs& a, cudaStream_t s) {
    // NX_FIELD_BACKWARD_PATH=simt forces the SIMT fp64 variant (validation of the
    // tensor-core path).
    static const bool force_simt = [] {
        const char* e = getenv("NX_FIELD_BACKWARD_PATH");
        return e && strcmp(e, "simt") == 0;
    }();
    if (!force_simt && field_backward_tc_supported(a.scene.field)) return launch_field_backward_tc(a, s);
    return launch_field_backward_simt(a, s);
}

}  // namespace nx
