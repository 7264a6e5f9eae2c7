// losses_backward (losses.cpp:107-238) on sm_100a: the per-pixel loss terms of a
// training step and the upstream gradients render_backward consumes.
//
//   image    (1 - w.dssim) L1 + w.dssim (1 - SSIM)/2 on final_img (losses.cpp:124-139):
//            SSIM with the reference's 11x11 Gaussian window (sigma 1.5), zero-padded
//            separable blurs and C1/C2 (ssim.cpp:10-151), forward and adjoint, fp64;
//   texture  mean |gt - weight-normalised buffered texture| over pixels with buffered
//            mass >= 1e-6 (losses.cpp:141-181);
//   alpha    mean (1 - buffered mass) (losses.cpp:183-195);
//   opacity  mean sigmoid(opacity_raw) -> grads.prims[i].opacity_raw (losses.cpp:201-210);
//   grid     sum_l s_l^-3 sum table^2 -> grads.field.table (losses.cpp:212-228).
// Every pixel term is one thread (per channel for SSIM); block partials meet in exact
// order-independent accumulators (nx_xacc.cuh), so the terms are bit-reproducible; a
// last kernel forms LossTerms on the device.
#include <algorithm>
#include <cmath>

#include "nx_internal.cuh"

namespace nx {

namespace {

constexpr int kWin = 11, kHalf = 5;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;
constexpr int kThreads = 256;
constexpr int kMaxLevels = 64;

// Sums accumulated by the kernels (device, zeroed per call).
enum { kSumSsim, kSumL1, kSumTex, kSumAlpha, kSumOpacity, kSumGrid0, kSumVals = kSumGrid0 + kMaxLevels };
struct LossSums {
    double tex_included;  // a count of pixels: exact in any order
    unsigned long long words[kSumVals * kXaccWordsTotal];
};
__device__ __forceinline__ Xacc sums_acc(LossSums* s) { return Xacc{s->words, kSumVals}; }

struct LossArgs {
    int W, H, K;
    int64_t n_prims;
    const float* final_img;
    const double* weights;
    const float* texture;
    const int32_t* ids;
    const double* gt;
    const double* geom;  // kGeomFields x n SoA (opacity_raw is field 9)
    const float* table;
    const double* table64;  // optional fp64 master of the table (nullptr: use `table`)
    int levels;
    int64_t level_entries;  // 2^log2 * features
    nx_loss_weights w;
    double* d_final;
    double* d_weights;
    double* d_texture;
    double* g_prims;
    double* g_table;
    nx_loss_terms* terms;
    LossSums* sums;
    double* maps;  // [3 ch][5] H-blurs, [3][3] SSIM partials, [3][3] their H-blurs
    double s3[kMaxLevels];  // pow(level_scale, 3) (losses.cpp:221)
};

__constant__ double c_taps[kWin];

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1)
        v += __hiloint2double(__shfl_xor_sync(0xffffffffu, __double2hiint(v), m),
                              __shfl_xor_sync(0xffffffffu, __double2loint(v), m));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += sh[i];
    return s;  // valid in thread 0
}

__device__ __forceinline__ double sgn(double v) { return v > 0 ? 1.0 : (v < 0 ? -1.0 : 0.0); }

// maps layout helpers
__device__ __forceinline__ double* hmap(const LossArgs& a, int c, int m) {  // 5 per channel
    return a.maps + (static_cast<int64_t>(c) * 5 + m) * a.W * a.H;
}
__device__ __forceinline__ double* dmap(const LossArgs& a, int c, int m) {  // 3 per channel
    return a.maps + (15 + static_cast<int64_t>(c) * 3 + m) * a.W * a.H;
}
__device__ __forceinline__ double* hdmap(const LossArgs& a, int c, int m) {
    return a.maps + (24 + static_cast<int64_t>(c) * 3 + m) * a.W * a.H;
}

// blur (ssim.cpp:31-57), horizontal half: x, y, x^2, y^2, xy of one channel
__global__ void __launch_bounds__(kThreads) ssim_hpass_kernel(const LossArgs a) {
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= npix) return;
    const int x = static_cast<int>(i % a.W);
    const int64_t row = i - x;
    const int k0 = max(-kHalf, -x), k1 = min(kHalf, a.W - 1 - x);
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = k0; k <= k1; ++k) {
        const double g = c_taps[k + kHalf];
        const double xv = static_cast<double>(a.final_img[(row + x + k) * 3 + c]);
        const double yv = a.gt[(row + x + k) * 3 + c];
        s[0] += g * xv;
        s[1] += g * yv;
        s[2] += g * (xv * xv);
        s[3] += g * (yv * yv);
        s[4] += g * (xv * yv);
    }
#pragma unroll
    for (int m = 0; m < 5; ++m) hmap(a, c, m)[i] = s[m];
}

// vertical half + the SSIM map and its partials wrt (mu_x, E[x^2], E[xy]) (ssim.cpp:126-141)
__global__ void __launch_bounds__(kThreads) ssim_vpass_kernel(const LossArgs a) {
    __shared__ double sh[kThreads / 32];
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    double s_val = 0.0;
    if (i < npix) {
        const int y = static_cast<int>(i / a.W);
        const int k0 = max(-kHalf, -y), k1 = min(kHalf, a.H - 1 - y);
        double b[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = k0; k <= k1; ++k) {
            const double g = c_taps[k + kHalf];
            const int64_t j = i + static_cast<int64_t>(k) * a.W;
#pragma unroll
            for (int m = 0; m < 5; ++m) b[m] += g * hmap(a, c, m)[j];
        }
        const double mx = b[0], my = b[1];
        const double sxx = b[2] - mx * mx, syy = b[3] - my * my, sxy = b[4] - mx * my;
        const double a1 = 2 * mx * my + kC1, a2 = 2 * sxy + kC2;
        const double b1 = mx * mx + my * my + kC1, b2 = sxx + syy + kC2;
        const double s = (a1 * a2) / (b1 * b2);
        s_val = s;
        const double scale = 1.0 / (3.0 * static_cast<double>(npix));
        dmap(a, c, 0)[i] = scale * ((2 * my * a2 - 2 * my * a1) / (b1 * b2) - s * (2 * mx / b1 - 2 * mx / b2));
        dmap(a, c, 1)[i] = scale * (-s / b2);
        dmap(a, c, 2)[i] = scale * (2 * a1 / (b1 * b2));
    }
    const double t = block_sum(s_val, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumSsim, t);
}

// adjoint blur, horizontal half, of the three partial maps
__global__ void __launch_bounds__(kThreads) ssim_bwd_hpass_kernel(const LossArgs a) {
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= npix) return;
    const int x = static_cast<int>(i % a.W);
    const int k0 = max(-kHalf, -x), k1 = min(kHalf, a.W - 1 - x);
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = k0; k <= k1; ++k) {
        const double g = c_taps[k + kHalf];
#pragma unroll
        for (int m = 0; m < 3; ++m) s[m] += g * dmap(a, c, m)[i + k];
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) hdmap(a, c, m)[i] = s[m];
}

// vertical half -> d SSIM / d pred (ssim.cpp:142-148), then the image-term gradient
// d_final = (1 - w) sign(pred - gt) / (3 n) - w/2 dSSIM (losses.cpp:130-136)
__global__ void __launch_bounds__(kThreads) ssim_bwd_vpass_kernel(const LossArgs a) {
    __shared__ double sh[kThreads / 32];
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    double l1 = 0.0;
    if (i < npix) {
        const int y = static_cast<int>(i / a.W);
        const int k0 = max(-kHalf, -y), k1 = min(kHalf, a.H - 1 - y);
        double b[3] = {0.0, 0.0, 0.0};
        for (int k = k0; k <= k1; ++k) {
            const double g = c_taps[k + kHalf];
            const int64_t j = i + static_cast<int64_t>(k) * a.W;
#pragma unroll
            for (int m = 0; m < 3; ++m) b[m] += g * hdmap(a, c, m)[j];
        }
        const double xv = static_cast<double>(a.final_img[i * 3 + c]), yv = a.gt[i * 3 + c];
        const double d_ssim = b[0] + 2 * xv * b[1] + yv * b[2];
        const double diff = xv - yv;
        l1 = fabs(diff);
        const double l1_scale = 1.0 / (3.0 * static_cast<double>(npix));
        a.d_final[i * 3 + c] = (1.0 - a.w.dssim) * sgn(diff) * l1_scale - 0.5 * a.w.dssim * d_ssim;
    }
    const double t = block_sum(l1, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumL1, t);
}

// texture supervision and coverage, pass 1: included count, texture error, coverage
__global__ void __launch_bounds__(kThreads) tex_alpha_sums_kernel(const LossArgs a) {
    __shared__ double sh[kThreads / 32];
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double inc = 0.0, err = 0.0, cov = 0.0;
    if (p < npix) {
        double sw = 0.0;
        for (int j = 0; j < a.K; ++j) sw += a.weights[p * a.K + j];
        cov = 1.0 - sw;
        if (sw >= 1e-6) {  // kTextureLossMinWeight (losses.hpp:30)
            inc = 1.0;
            for (int c = 0; c < 3; ++c) {
                double r = 0.0;
                for (int j = 0; j < a.K; ++j) r += a.weights[p * a.K + j] * a.texture[(p * a.K + j) * 3 + c];
                err += fabs(a.gt[p * 3 + c] - r / sw);
            }
        }
    }
    const double s0 = block_sum(inc, sh);
    if (threadIdx.x == 0 && s0 != 0.0) atomicAdd(&a.sums->tex_included, s0);
    const double s1 = block_sum(err, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumTex, s1);
    const double s2 = block_sum(cov, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumAlpha, s2);
}

// pass 2: d_texture and d_weights of every slot (overwritten)
__global__ void __launch_bounds__(kThreads) tex_alpha_grad_kernel(const LossArgs a) {
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    const double included = a.sums->tex_included;
    const double coef = included > 0 ? a.w.texture / (3.0 * included) : 0.0;
    const double a_coef = a.w.alpha / static_cast<double>(npix);
    double sw = 0.0;
    for (int j = 0; j < a.K; ++j) sw += a.weights[p * a.K + j];
    const bool inc = sw >= 1e-6 && included > 0;
    double rn[3] = {0.0, 0.0, 0.0};
    if (inc)
        for (int c = 0; c < 3; ++c) {
            double r = 0.0;
            for (int j = 0; j < a.K; ++j) r += a.weights[p * a.K + j] * a.texture[(p * a.K + j) * 3 + c];
            rn[c] = r / sw;
        }
    for (int j = 0; j < a.K; ++j) {
        const int64_t sl = p * a.K + j;
        double dw = 0.0, dt[3] = {0.0, 0.0, 0.0};
        if (a.ids[sl] >= 0) {
            if (inc) {
                double dw_acc = 0.0;
                for (int c = 0; c < 3; ++c) {
                    const double sg = sgn(rn[c] - a.gt[p * 3 + c]);
                    dt[c] = coef * sg * a.weights[sl] / sw;
                    dw_acc += sg * (static_cast<double>(a.texture[sl * 3 + c]) - rn[c]);
                }
                dw = coef * dw_acc / sw;
            }
            dw -= a_coef;
        }
        a.d_weights[sl] = dw;
        a.d_texture[sl * 3 + 0] = dt[0];
        a.d_texture[sl * 3 + 1] = dt[1];
        a.d_texture[sl * 3 + 2] = dt[2];
    }
}

// opacity regulariser (losses.cpp:201-210)
__global__ void __launch_bounds__(kThreads) opacity_kernel(const LossArgs a) {
    __shared__ double sh[kThreads / 32];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double o = 0.0;
    if (i < a.n_prims) {
        o = sigmoid(a.geom[9 * a.n_prims + i]);
        a.g_prims[i * NX_PARAMS_PER_NEXEL + 9] += (a.w.opacity / static_cast<double>(a.n_prims)) * o * (1.0 - o);
    }
    const double t = block_sum(o, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumOpacity, t);
}

// grid regulariser (losses.cpp:212-228): one level slab per blockIdx.y
__global__ void __launch_bounds__(kThreads) grid_kernel(const LossArgs a) {
    __shared__ double sh[kThreads / 32];
    const int l = blockIdx.y;
    const double s3 = a.s3[l];
    const int64_t base = static_cast<int64_t>(l) * a.level_entries;
    double acc = 0.0;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < a.level_entries;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // the fp64 master of the table when the trainer keeps one (the values being
        // optimised), else the scene's fp32 render copy
        const double v = a.table64 ? a.table64[base + e] : static_cast<double>(a.table[base + e]);
        acc += v * v;
        a.g_table[base + e] += a.w.grid * 2.0 * v / s3;
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) xacc_add(sums_acc(a.sums), kSumGrid0 + l, t);
}

// LossTerms (losses.cpp:137-139, 162, 195, 209, 227, 231-232)
__global__ void terms_kernel(const LossArgs a) {
    const Xacc acc = sums_acc(a.sums);
    const double tex_included = a.sums->tex_included;
    const double s_ssim = xacc_take(acc, kSumSsim), s_l1 = xacc_take(acc, kSumL1), s_tex = xacc_take(acc, kSumTex),
                 s_alpha = xacc_take(acc, kSumAlpha), s_opacity = xacc_take(acc, kSumOpacity);
    const double npix = static_cast<double>(a.W) * a.H;
    nx_loss_terms t;
    t.l1 = s_l1 / (3.0 * npix);
    t.dssim = (1.0 - s_ssim / (3.0 * npix)) / 2.0;
    t.image = (1.0 - a.w.dssim) * t.l1 + a.w.dssim * t.dssim;
    if (a.K > 0) {
        t.texture = tex_included > 0 ? s_tex / (3.0 * tex_included) : 0.0;
        t.alpha = s_alpha / npix;
    } else {
        t.texture = 0.0;
        t.alpha = 1.0;
    }
    t.opacity = a.n_prims > 0 ? s_opacity / static_cast<double>(a.n_prims) : 0.0;
    double g = 0.0;
    for (int l = 0; l < a.levels; ++l) g += xacc_take(acc, kSumGrid0 + l) / a.s3[l];
    t.grid = g;
    t.total = t.image + a.w.texture * t.texture + a.w.alpha * t.alpha + a.w.opacity * t.opacity + a.w.grid * t.grid;
    *a.terms = t;
}

__global__ void pixel_error_kernel(const float* __restrict__ final_img, const double* __restrict__ gt, int64_t npix,
                                   double* __restrict__ err) {
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    double e = 0.0;
    for (int c = 0; c < 3; ++c) e += fabs(static_cast<double>(final_img[p * 3 + c]) - gt[p * 3 + c]);
    err[p] = e / 3.0;
}

}  // namespace

void launch_pixel_error(const float* final_img, const double* gt, int64_t npix, double* err, cudaStream_t s) {
    if (npix <= 0) return;
    count_launch();
    pixel_error_kernel<<<static_cast<unsigned>((npix + kThreads - 1) / kThreads), kThreads, 0, s>>>(final_img, gt,
                                                                                                   npix, err);
}

size_t losses_scratch_bytes(int64_t npix) { return sizeof(LossSums) + 256 + static_cast<size_t>(33) * npix * sizeof(double); }

int launch_losses_backward(const SceneDev& scene, const FrameDev& fb, const double* gt, const nx_loss_weights& w,
                           double* d_final, double* d_weights, double* d_texture, double* g_prims, double* g_table,
                           nx_loss_terms* terms, void* scratch, cudaStream_t s, const double* table64) {
    if (scene.field.levels > kMaxLevels) return NX_UNSUPPORTED;
    static uint64_t taps_ready = 0;  // per device: __constant__ memory is per device
    int cur = 0;
    cudaGetDevice(&cur);
    if (!((taps_ready >> (cur & 63)) & 1)) {  // gaussian_taps (ssim.cpp:15-28)
        double t[kWin], sum = 0.0;
        for (int i = 0; i < kWin; ++i) {
            const double d = i - kHalf;
            t[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += t[i];
        }
        for (double& v : t) v /= sum;
        if (cudaMemcpyToSymbol(c_taps, t, sizeof t) != cudaSuccess) return NX_CUDA_ERROR;
        taps_ready |= uint64_t(1) << (cur & 63);
    }
    LossArgs a;
    a.W = fb.W;
    a.H = fb.H;
    a.K = fb.K;
    a.n_prims = scene.n;
    a.final_img = fb.final_img;
    a.weights = fb.weights;
    a.texture = fb.texture;
    a.ids = fb.ids;
    a.gt = gt;
    a.geom = scene.geom;
    a.table = scene.table;
    a.table64 = table64;
    a.levels = scene.field.levels;
    a.level_entries = (int64_t(1) << scene.field.log2_table) * scene.field.features;
    a.w = w;
    a.d_final = d_final;
    a.d_weights = d_weights;
    a.d_texture = d_texture;
    a.g_prims = g_prims;
    a.g_table = g_table;
    a.terms = terms;
    a.sums = static_cast<LossSums*>(scratch);
    a.maps = reinterpret_cast<double*>(static_cast<char*>(scratch) + ((sizeof(LossSums) + 255) / 256) * 256);
    double sc = scene.field.base_scale;
    for (int l = 0; l < a.levels; ++l, sc *= scene.field.growth) a.s3[l] = std::pow(sc, 3.0);
    const int64_t npix = static_cast<int64_t>(a.W) * a.H;
    if (cudaMemsetAsync(a.sums, 0, sizeof(LossSums), s) != cudaSuccess) return NX_CUDA_ERROR;
    if (npix > 0) {
        const dim3 g3(static_cast<unsigned>((npix + kThreads - 1) / kThreads), 3);
        const unsigned g1 = static_cast<unsigned>((npix + kThreads - 1) / kThreads);
        count_launch(4);
        ssim_hpass_kernel<<<g3, kThreads, 0, s>>>(a);
        ssim_vpass_kernel<<<g3, kThreads, 0, s>>>(a);
        ssim_bwd_hpass_kernel<<<g3, kThreads, 0, s>>>(a);
        ssim_bwd_vpass_kernel<<<g3, kThreads, 0, s>>>(a);
        if (a.K > 0) {
            count_launch(2);
            tex_alpha_sums_kernel<<<g1, kThreads, 0, s>>>(a);
            tex_alpha_grad_kernel<<<g1, kThreads, 0, s>>>(a);
        }
    }
    if (a.n_prims > 0) {
        count_launch();
        opacity_kernel<<<static_cast<unsigned>((a.n_prims + kThreads - 1) / kThreads), kThreads, 0, s>>>(a);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>((a.level_entries + kThreads - 1) / kThreads,
                                                                std::max(1, 2 * sms / std::max(1, a.levels)) * 4));
    count_launch(2);
    grid_kernel<<<dim3(gx, a.levels), kThreads, 0, s>>>(a);
    terms_kernel<<<1, 1, 0, s>>>(a);
    return NX_OK;
}

}  // namespace nx
