// Internal declarations shared by the sm_100a render kernels.
//
// Device-side fp64 restatements of the reference math the render path makes
// decisions with. Every discrete decision of the reference (cull, straddle,
// tile rect, (depth,id) order, grazing / near-plane / 1/255 tests, alpha clamp,
// termination, top-K) is taken in fp64 with the reference's formulas, so the
// discrete outputs (tile lists, contributor lists, ids) are bit-exact.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/nexel_b200.h"
#include "nx_xacc.cuh"

#define NX_HD __host__ __device__ __forceinline__

namespace nx {

constexpr double kAlphaMin = 1.0 / 255.0;  // kernel.hpp:11
constexpr double kMinNormalDot = 1e-8;     // intersect.hpp:12
constexpr double kProjectMinDepth = 1e-9;  // camera.hpp:38
constexpr int kMaxTopK = NX_MAX_TOP_K;
constexpr int kGeomFields = 12;            // fp64 geometry params per primitive
// Work lists are built per 8x8 pixel tile (the composite's CTA), independent of
// settings.tile: every hit of a primitive lies inside its padded pixel rect, so the
// per-pixel contributor sequences do not depend on the list granularity.
constexpr int kWorkTile = 8;
// The reverse march (render_backward) walks 16x16-pixel work lists: its CTAs are
// 8 warps that share per-primitive gradient accumulators in shared memory.
constexpr int kBwdTile = 8;  // render_backward work tiles (the forward's; 16 selectable)

// ---------------------------------------------------------------- scalar helpers
// sigmoid / softplus (vec_math.hpp:69-84)
NX_HD double sigmoid(double x) {
    if (x >= 0) {
        const double e = exp(-x);
        return 1.0 / (1.0 + e);
    }
    const double e = exp(x);
    return e / (1.0 + e);
}
NX_HD double softplus(double x) {
    if (x > 30.0) return x;
    if (x < -30.0) return exp(x);
    return log1p(exp(x));
}
// axis_power / eval_kernel / support_radius (kernel.hpp:16-30, 72-76)
NX_HD double axis_power(double u, double g) {
    if (u == 0.0) return 0.0;
    if (g == 1.0) return u * u;
    const double e = 2.0 * g * log(fabs(u));
    if (e > 700.0) return INFINITY;
    return exp(e);
}
// axis_power with log|u| supplied (the same value axis_power forms, so bit-identical)
NX_HD double axis_power_log(double u, double g, double lu) {
    if (u == 0.0) return 0.0;
    if (g == 1.0) return u * u;
    const double e = 2.0 * g * lu;
    if (e > 700.0) return INFINITY;
    return exp(e);
}
NX_HD double eval_kernel(double u, double v, double o, double gx, double gy) {
    const double p = axis_power(u, gx) + axis_power(v, gy);
    if (isinf(p)) return 0.0;
    return o * exp(-0.5 * p);
}
// pow(lim, 1/(2g)) as exp(log(lim) / (2g)): |log(lim)/(2g)| <= ~1 here, so the
// result stays within a few ulp of the reference's glibc pow (rect decisions have
// >= 1e-9 relative margin) at a fraction of pow's cost.
NX_HD double support_radius(double o, double g) {
    const double lim = 2.0 * log(o / kAlphaMin);
    if (lim <= 0.0) return 0.0;
    return exp(log(lim) / (2.0 * g));
}
// static_cast<int>(floor(x)) with x86 cvttsd2si semantics (out-of-range -> INT_MIN),
// which is what the reference's casts produce on its host (renderer.cpp:84-87).
NX_HD int x86_to_int(double v) {
    if (v >= -2147483648.0 && v < 2147483648.0) return static_cast<int>(v);
    return INT32_MIN;
}
NX_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

// Orderable 64-bit key for a finite double; -0.0 is canonicalised to +0.0 so
// that equal depths tie (and fall back to id order, renderer.cpp:102-105).
NX_HD uint64_t depth_key(double d) {
    d = d + 0.0;
#ifdef __CUDA_ARCH__
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t b;
    memcpy(&b, &d, 8);
#endif
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ---------------------------------------------------------------- camera (camera.hpp:17-43)
struct CamD {
    int W, H;
    double fx, fy, cx, cy;
    double R[9];  // row-major
    double t[3];
    double o[3];  // position() = -R^T t
};

// pixel_ray (camera.hpp:32-35): dir = R^T normalized(((px-cx)/fx, (py-cy)/fy, 1)).
NX_HD void pixel_dir(const CamD& c, double px, double py, double* dir) {
    const double d0 = (px - c.cx) / c.fx, d1 = (py - c.cy) / c.fy, d2 = 1.0;
    const double n = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    const double n0 = d0 / n, n1 = d1 / n, n2 = d2 / n;
    dir[0] = c.R[0] * n0 + c.R[3] * n1 + c.R[6] * n2;
    dir[1] = c.R[1] * n0 + c.R[4] * n1 + c.R[7] * n2;
    dir[2] = c.R[2] * n0 + c.R[5] * n1 + c.R[8] * n2;
}

// ---------------------------------------------------------------- per-primitive composite record
// AoS, 24 fp64 per primitive (192 B), staged into shared memory by the compositing kernels.
enum RecField {
    REC_NUM = 0,  // dot(mu - origin, n): the per-camera numerator of t (intersect.hpp:29)
    REC_NX, REC_NY, REC_NZ,
    REC_V1X, REC_V1Y, REC_V1Z,
    REC_V2X, REC_V2Y, REC_V2Z,
    REC_MUX, REC_MUY, REC_MUZ,
    REC_SX, REC_SY,
    REC_OP,
    REC_GX, REC_GY,
    REC_ULIM, REC_VLIM,  // conservative |dot(delta,v)| bounds for an exact early reject
    REC_RSX, REC_RSY,    // 1 / sigma (the certified fp32 alpha, nx_fastmath.cuh cert_alpha)
    REC_OM,              // 1 - opacity = sigmoid(-opacity_raw), for an accurate 1 - alpha
    REC_PAD,
    REC_FIELDS
};

// Classification of a primitive by build_binning (renderer.cpp:52-100).
enum PrimClass : int32_t {
    CLS_SUPPORT = 0,    // ru <= 0 || rv <= 0, no entry
    CLS_BEHIND = 1,     // whole support behind the pinhole, no entry
    CLS_OFFSCREEN = 2,  // rect entirely off screen, no entry
    CLS_RECT = 3,       // rect-binned entry
    CLS_STRADDLER = 4,  // entry in every tile (reference); refined work rect here
};

// Near-threshold decisions (the safety net of the bit-exact claim): decisions taken in
// fp64 with the reference's formulas whose margin is below a generous bound (>= 100x)
// on the error the device math can have against the reference's (its own exp / log
// routines instead of glibc's, exp(log / 2g) instead of pow, FMA contraction). Zero in
// the parity tests; reported by the bench.
enum NearKind { NEAR_ALPHA = 0, NEAR_TRANSMITTANCE, NEAR_TOPK, NEAR_DEPTH, NEAR_RECT, NEAR_SUPPORT, NEAR_KINDS };
constexpr double kNearRel = 1e-11;        // T and top-K weights (products over up to ~100 hits)
constexpr double kNearAlpha = 1e-12;      // alpha vs 1/255 (exp of a sum of powers: ~1e-14)
constexpr double kNearDepth = 1e-13;      // camera-z of mu: a 3-term dot product + add (~4 ulp)
constexpr double kNearPixel = 1e-9;       // rect floor / ceil arguments, in pixels (~1e-12 px)
constexpr double kNearSupport = 1e-13;    // 2 ln(255 o) vs 0

struct FrameStatsD {
    unsigned long long cls[5];
    unsigned long long straddlers_kept;
    unsigned long long tile_keys;
    unsigned long long work_keys;
    unsigned long long queries;
    unsigned long long near[NEAR_KINDS];
    unsigned long long redo_tiles;  // pixels the certified composite handed to the exact redo
};

struct SceneDev {
    int64_t n;
    const double* geom;  // kGeomFields x n SoA: mu xyz, quat wxyz, log_scale xy, opacity_raw, gamma_raw xy
    const float* sh;     // n x 48 (coefficient-major, rgb interleaved), fp32
    const float* table;  // levels x 2^log2 x features, fp32
    const float* w1;     // hidden x n_in
    const float* w2;     // hidden x hidden
    const float* w3;     // 48 x hidden
    nx_field_desc field;
    // NX_PRECISION_F64 scenes: fp64 copies of the colour inputs (else nullptr)
    const double* sh64 = nullptr;
    const double* table64 = nullptr;
    const double* w1_64 = nullptr;
    const double* w2_64 = nullptr;
    const double* w3_64 = nullptr;
};

struct FrameDev {
    int W, H, K, tiles_x, tiles_y;
    float* base;
    int32_t* ids;
    double* depths;
    double* weights;
    float* texture;
    float* final_img;
    float* residual;
    double* residual64;  // fp64 terminal transmittance (nullptr unless the frame keeps backward state)
    double* base64;  // optional fp64 base (backward state), nullptr if not kept
    double* texture64 = nullptr;  // NX_PRECISION_F64: fp64 texture / final
    double* final64 = nullptr;
};

// Host-side count of kernel launches issued by this library (all contexts).
void count_launch(int n = 1);

// ---------------------------------------------------------------- launchers
struct PreprocessArgs {
    SceneDev scene;
    nx_settings st;
    CamD cam;
    int tiles_x, tiles_y;  // reference tiles (settings.tile)
    int work_tile;         // pixel size of the work-list tiles (kWorkTile)
    double zmin_work;   // conservative camera-z bound of any hit (straddler refinement)
    double* rec;        // n x REC_FIELDS (AoS, 160 B per primitive)
    float4* recf;       // n x 4 fp32 prefilter records (64 B per primitive)
    int32_t* cls;       // n
    int4* ref_rect;     // n
    int4* work_rect;    // n
    uint64_t* key;      // n
    int32_t* flag;      // n: 1 if the primitive enters the sort (work or reference mode)
    int reference_lists;
    FrameStatsD* stats;
};
void launch_preprocess(const PreprocessArgs& a, cudaStream_t s);

// activate()'s validation (primitive.cpp:47-63) of a device scene: *first (preset to
// ~0) receives min(id * 8 + check) over the failing primitives.
void launch_validate(const double* geom, const float* sh, int64_t n, unsigned long long* first, cudaStream_t s);

// Gathers (key, id) of flagged primitives at their scanned positions (id-ascending).
void launch_compact(const int32_t* flag, const int32_t* pos, const uint64_t* key, int64_t n,
                    uint64_t* keys_out, uint32_t* ids_out, cudaStream_t s);

// counts[r] = tiles of rect[ids[r]] (work or reference rect) for r < *n_dev, 0 up to n.
// (+ counts sorted neighbours whose depths differ by less than kNearRel: NEAR_DEPTH)
void launch_rect_counts(const uint32_t* ids, int64_t n, const int32_t* n_dev, const int4* rect, int32_t* counts,
                        const uint64_t* sorted_keys, FrameStatsD* stats, cudaStream_t s);

// Emits (tile, id) for every tile of every sorted primitive's rect, in sorted
// order (row-major tiles, renderer.cpp:106-110), and counts keys per tile. The sorted
// count and key count are read on the device (*n_sorted_dev, *n_keys_dev); keys past
// the capacity key_cap are not written (nor counted).
// The work-list cull of emit (tiles whose corner rays' support quadrilateral misses):
// recf == nullptr disables it (reference lists stay the reference's).
struct EmitCull {
    const float4* recf = nullptr;
    int n_tiles = 0, tiles_x = 0, tile = 8, W = 0, H = 0;
    float cx = 0.f, cy = 0.f, ifx = 1.f, ify = 1.f;
    float R[9] = {};
};
void launch_emit(const uint32_t* ids, const int32_t* offsets, int64_t sorted_cap, const int32_t* n_sorted_dev,
                 int64_t key_cap, const int32_t* n_keys_dev, const int4* rect, int tiles_x, uint32_t* tile_keys,
                 uint32_t* vals, int32_t* tile_counts, const EmitCull& cull, cudaStream_t s);

struct CompositeArgs {
    const double* rec;   // n x REC_FIELDS
    const float4* recf;  // n x 4
    int64_t n;
    const float* sh;
    const int32_t* list_ids;
    const int32_t* tile_offsets;
    nx_settings st;
    CamD cam;
    FrameDev fb;
    int sh_degree;
    int32_t* dbg_hits;   // optional: per-pixel hit ids (rows [dbg_y0, dbg_y1))
    int32_t* dbg_counts;
    int dbg_y0, dbg_y1, dbg_max;
    FrameStatsD* stats;  // near-threshold counters
    const double* sh64 = nullptr;  // NX_PRECISION_F64: fp64 SH (the colour path runs in fp64)
    // certified fp32 alpha (nx_fastmath.cuh cert_alpha) for frames without backward state:
    // the first pass appends the pixels it could not certify to redo ([0] = count, zeroed
    // by the caller), a warp-per-pixel exact pass re-renders them
    bool certified = false;
    bool redo_all = false;  // tests: hand every pixel to the exact redo
    int32_t* redo = nullptr;
};
void launch_composite(const CompositeArgs& a, cudaStream_t s);

struct TextureArgs {
    SceneDev scene;
    nx_settings st;
    CamD cam;
    FrameDev fb;
    FrameStatsD* stats;
    float* fscratch;  // H*W*K*32 interpolated features (split tensor-core path), per frame
    cudaEvent_t ev_mid = nullptr;          // profiling: recorded between the gathers and the decoder
    mutable bool ev_mid_recorded = false;  // set by the launcher when it recorded ev_mid
};
int launch_texture(const TextureArgs& a, cudaStream_t s);  // returns NX_OK / NX_UNSUPPORTED
// tcgen05 variant for the reference field shape (16 levels x 2 features, 64 hidden).
bool texture_tc_supported(const nx_field_desc& fd);
// 0: warp-specialised with gather warps, 1: fused single-role, 2: split (gathers, then
// the MLP over an fp32 feature scratch), 3: bulk-fed warp-specialised (gathers into
// pre-split operand tiles, then the MMA pipeline fed by cp.async.bulk), 4: split2
// (gathers into pre-split operand tiles, then a single-role decoder that double-buffers
// them with cp.async.bulk), 5: split2ts (default: split2 with the decoder's hidden
// activations in tensor memory, three CTAs per SM)
int texture_tc_path();
// bytes of TextureArgs::fscratch the selected path needs for a W x H x K frame (0: none)
size_t texture_tc_scratch_bytes(int W, int H, int K);
int launch_texture_tc(const TextureArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- losses_backward (nx_losses.cu)
size_t losses_scratch_bytes(int64_t npix);
int launch_losses_backward(const SceneDev& scene, const FrameDev& fb, const double* gt, const nx_loss_weights& w,
                           double* d_final, double* d_weights, double* d_texture, double* g_prims, double* g_table,
                           nx_loss_terms* terms, void* scratch, cudaStream_t s, const double* table64 = nullptr);

// ---------------------------------------------------------------- Adam (nx_adam.cu)
void adam_group_sizes(const SceneDev& sc, int64_t* sizes);
// master: the group's fp64 master values (groups 5..10; nullptr: step the fp32 values)
void launch_adam_group(int group, const SceneDev& sc, double* geom, float* sh, float* table, float* w1, float* w2,
                       float* w3, const nx_grads& g, double* m, double* v, double* master, const nx_adam_config& cfg,
                       int64_t step, cudaStream_t s);
// a group's values <-> its row layout (rows: device, the group's size)
void launch_group_io(int group, const SceneDev& sc, double* geom, float* sh, float* table, float* w1, float* w2,
                     float* w3, double* rows, bool to_rows, cudaStream_t s);
// err[p] = sum_c |final - gt| / 3 (trainer.cpp:288-295)
void launch_pixel_error(const float* final_img, const double* gt, int64_t npix, double* err, cudaStream_t s);

// ---------------------------------------------------------------- density control (nx_density.cu)
void launch_prune_flags(const double* geom, int64_t n, double min_opacity, int32_t* flags, cudaStream_t s);
void launch_compact_map(const int32_t* flags, const int32_t* pos, int64_t n, int32_t* n2o, cudaStream_t s);
void launch_gather_geom(const double* geom, int64_t n, double* out, int64_t n_new, const int32_t* n2o, cudaStream_t s);
void launch_gather_rows_f32(const float* in, float* out, int64_t n_new, int width, const int32_t* n2o, cudaStream_t s);
void launch_gather_rows_f64(const double* in, double* out, int64_t n_new, int width, const int32_t* n2o,
                            cudaStream_t s);
void launch_split_keys(const double* errors, const double* uniforms, int64_t n, uint64_t* keys, uint32_t* ids,
                       unsigned long long* n_keys, cudaStream_t s);
void launch_split_children(double* geom_new, int64_t n_new, const double* geom_old, int64_t n, float* sh,
                           const int32_t* parents, int64_t count, int32_t* n2o, cudaStream_t s);

// ---------------------------------------------------------------- downloads
struct CopyJob {
    const uint8_t* src;  // device
    uint8_t* dst;        // device-mapped pinned host memory
    size_t bytes;        // source bytes
    int narrow;          // 1: src is fp64, dst receives it as fp32 (bytes / 2)
};
struct CopyJobs {
    CopyJob j[8];
    int n;
};
// Streaming (evict-first) device -> mapped-host copy of up to 8 buffers (nx_copy.cu).
void launch_stream_copy(const CopyJobs& jobs, cudaStream_t s);

// ---------------------------------------------------------------- backward (render_backward)
// Per-primitive activated-space gradient accumulator (ActivatedGrad,
// intersect.hpp:45-51) + the blended-error sum: d_mu[3], d_R[9] (row-major m[i][j],
// columns v1, v2, n), d_sigma[2], d_opacity, d_gamma[2], blended error.
constexpr int kActFields = 18;
// Exact per-primitive accumulator values of the compositing branch: the activated
// fields + the 48 SH gradients (nx_xacc.cuh).
constexpr int kPrimAccVals = kActFields + NX_SH_VALUES;

// Device scratch of the field backward, owned by the context (grow-only; the exact
// accumulators are zeroed when allocated and kept zero between calls by their readers).
struct FieldBwdScratch {
    float* fbuf = nullptr;
    size_t fcap = 0;
    int32_t* amb = nullptr;
    size_t acap = 0;
    unsigned long long* tx = nullptr;  // table-gradient accumulators (nx_xacc.cuh)
    size_t txcap = 0;                  // bytes
    unsigned long long* wx = nullptr;  // MLP weight-gradient accumulators (SIMT path)
    size_t wxcap = 0;
    float* parts = nullptr;
    size_t pcap = 0;
    float* jbuf = nullptr;  // per-slot level sums (features pass -> scatter)
    size_t jcap = 0;
    static int grow_zeroed(unsigned long long*& p, size_t& cap, size_t bytes, cudaStream_t s) {
        if (bytes <= cap && p) return NX_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return NX_OUT_OF_MEMORY;
        if (cudaMemsetAsync(p, 0, bytes, s) != cudaSuccess) return NX_CUDA_ERROR;
        cap = bytes;
        return NX_OK;
    }
    int table_acc(int64_t m, cudaStream_t s) { return grow_zeroed(tx, txcap, xacc_bytes(m), s); }
    int weight_acc(int64_t m, cudaStream_t s) { return grow_zeroed(wx, wxcap, xacc_bytes(m), s); }
    void release() {
        for (void* p : {static_cast<void*>(fbuf), static_cast<void*>(amb), static_cast<void*>(tx),
                        static_cast<void*>(wx), static_cast<void*>(parts), static_cast<void*>(jbuf)})
            if (p) cudaFree(p);
        *this = FieldBwdScratch{};
    }
};
// g += the accumulators' sums, zeroing them (nx_field_backward_tc.cu)
__global__ void take_table_kernel(double* __restrict__ g, const Xacc acc);

struct FieldBwdArgs {
    SceneDev scene;
    nx_settings st;
    CamD cam;
    FrameDev fb;
    const double* d_final;    // H*W*3 or nullptr
    const double* d_texture;  // H*W*K*3 or nullptr
    double* d_t_slot;         // H*W*K out: dL/dt of each buffered crossing (0 for empty slots)
    double* g_table;          // levels * 2^log2 * features (accumulated)
    double* g_w1;
    double* g_w2;
    double* g_w3;
    FieldBwdScratch* scratch;  // the context's
    // optional: the table-gradient scatter runs on `side` (forked after d_t_slot with
    // ev_fork); ev_join is recorded there when it is done (the caller joins it)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
// field_backward_batch (texture_field.cpp:77-146) over the buffered slots.
int launch_field_backward(const FieldBwdArgs& a, cudaStream_t s);
int launch_field_backward_simt(const FieldBwdArgs& a, cudaStream_t s);
bool field_backward_tc_supported(const nx_field_desc& fd);
int launch_field_backward_tc(const FieldBwdArgs& a, cudaStream_t s);

struct CompositeBwdArgs {
    const double* rec;
    const float4* recf;
    int64_t n;
    const float* sh;
    const int32_t* list_ids;
    const int32_t* tile_offsets;
    nx_settings st;
    CamD cam;
    FrameDev fb;
    int sh_degree;
    const double* d_final;    // H*W*3 or nullptr
    const double* d_weights;  // H*W*K or nullptr
    const double* d_t_slot;   // H*W*K
    const double* err_pixel;  // H*W or nullptr
    Xacc acc;                 // n x kPrimAccVals exact accumulators (zero on entry)
    int tile;                 // work-tile side of the lists: 16, or 8 for small images
};
// The per-pixel reverse march of render_backward (renderer.cpp:287-390).
void launch_composite_backward(const CompositeBwdArgs& a, cudaStream_t s);
// activation_backward (intersect.hpp:91-103) of the summed activated gradients.
// Reads the accumulators back (zeroing them) into act_grad / the SH gradients, then
// applies activation_backward.
void launch_prim_finalize(const SceneDev& scene, int no_gamma, const Xacc& acc, double* act_grad, double* prim_grad,
                          double* blended_error, cudaStream_t s);

}  // namespace nx
