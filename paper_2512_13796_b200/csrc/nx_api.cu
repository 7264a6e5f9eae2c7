// C-ABI of the B200 render path (include/nexel_b200.h) and the per-frame
// orchestration of the stages:
//
//   K1 preprocess ........ activation, projection, classification, rects, records
//   K2 depth sort ......... compaction + stable LSD radix sort of 64-bit depth keys
//   K3 emit ............... (tile, id) keys in sorted order + per-tile counts
//   K4 tile sort .......... stable LSD radix sort by tile -> front-to-back tile lists
//   K5 tile ranges ........ exclusive scan of per-tile counts
//   K6 composite .......... per-tile compositing, top-K, Eq. 6 base
//   K7 texture ............ hash grid + MLP + SH at the buffered crossings, Eq. 7
//
// Error behaviour follows the reference (renderer.cpp:116-117): settings are
// validated first (bad-settings), then the camera (bad-camera), then the
// primitives (bad-primitive, first failing id, as activate_all would throw).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "nx_internal.cuh"
#include "nx_nexl.h"
#include "nx_sort.cuh"

using namespace nx;

namespace nx {
void count_launch(int n);
}

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    // for exact accumulators (nx_xacc.cuh): a fresh allocation is zeroed; readers keep it zero
    cudaError_t ensure_zeroed(size_t bytes, cudaStream_t s) {
        if (bytes <= cap && p) return cudaSuccess;
        cudaError_t e = ensure(bytes);
        if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, cap, s);
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

std::atomic<unsigned long long> g_launches{0};

const char* kStageNames[NX_NUM_STAGES] = {"preprocess", "depth_sort", "emit",   "tile_sort",
                                          "composite",  "texture",    "texture_mlp"};

// Profiling event points per frame (stage k spans two points; the texture pass may
// run on the second stream, so it has its own start/end points).
enum EvPoint { kEvPre, kEvDepth, kEvEmit, kEvTileSort, kEvComp, kEvCompEnd, kEvTex, kEvTexMid, kEvTexEnd, kEvPoints };
constexpr int kEvSets = 4;

}  // namespace

void nx::count_launch(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed); }

struct nx_ctx {
    int device = 0;
    int sms = 148;  // multiprocessors of the device
    cudaStream_t stream = nullptr;
    std::string err;
    int err_status = NX_OK;
    // per-frame scratch (grow-only)
    DevBuf rec, recf, cls, ref_rect, work_rect, key, flag, pos;
    DevBuf skeys_a, skeys_b, sids_a, sids_b, counts, offsets;
    DevBuf tkeys_a, tkeys_b, tvals_a, tvals_b, tile_counts, scratch;
    DevBuf dbg_hits, dbg_counts;
    DevBuf redo;          // tiles the certified composite hands to the exact pass
    bool certified = true;  // NX_CERTIFIED=0: every frame on the exact fp64 composite
    bool redo_all = false;  // NX_CERT_REDO_ALL=1 (tests): every tile through the exact redo pass
    DevBuf valid_word;  // revalidation result (first failing primitive)
    // render_backward scratch
    nx_frame* bwd_lists = nullptr;   // work lists of the re-binned camera
    DevBuf d_t_slot, act_grad, xacc_prims;
    DevBuf dens_map, dens_par, dens_src;  // density-control maps (grow-only)
    // provenance of the work lists / records in the shared buffers (rec, recf, tile keys):
    // render_backward reuses a forward's lists when nothing rebuilt them since
    uint64_t lists_gen = 0;
    const nx_scene* lists_scene = nullptr;
    uint64_t lists_scene_version = 0;
    nx_camera lists_cam{};
    int lists_tile = 0;
    DevBuf h_up[3], h_err, h_blend, h_grads[5];  // device copies for nx_render_backward_host
    DevBuf loss_scratch, h_gt, h_terms;          // losses_backward
    FieldBwdScratch field_bwd;                    // tensor-core field backward
    int32_t* h_pinned = nullptr;  // small readbacks
    // Work-list key capacity of the asynchronous list builds (grow-only): sized from the
    // first frame's count (one synchronous build) and from the counts later frames report
    // back (asynchronously, nx_frame::h_counts); a frame that exceeded it is re-rendered
    // when it is first read back (frame_settle).
    int64_t key_cap = 0;
    bool sync_lists = false;  // NX_SYNC_LISTS=1: size every build from its own count (host round trip)
    bool emit_cull = true;    // NX_EMIT_CULL=0: keep every work-rect key (no corner-ray cull)
    bool profiling = false;
    cudaStream_t stream2 = nullptr;  // texture passes: overlap the next frame's collection
    cudaStream_t stream3 = nullptr;  // downloads: the copy engine overlaps both
    cudaEvent_t ev_join = nullptr;
    // render_backward: the table-gradient scatter beside the compositing backward
    // (forked and joined back inside each call)
    cudaStream_t stream_bwd = nullptr;
    cudaEvent_t ev_bwd_fork = nullptr, ev_bwd_join = nullptr;
    cudaEvent_t ev[kEvSets][kEvPoints] = {};
    int ev_cur = 0;
    bool ev_pending[kEvSets] = {};  // profiled frames whose events are not folded yet
    double stage_acc[NX_NUM_STAGES] = {};
    int stage_frames = 0;
};

// Scene versions are unique across scenes (a new scene may reuse a freed one's address).
uint64_t next_scene_version() {
    static std::atomic<uint64_t> v{0};
    return ++v;
}

struct nx_scene {
    nx_ctx* ctx = nullptr;
    int device = 0;  // the creating context's device (destroy must not touch a freed ctx)
    int64_t n = 0;
    DevBuf geom, sh, table, w1, w2, w3;
    DevBuf geom_spare, sh_spare;  // density control rebuilds into these and swaps (grow-only)
    DevBuf sh64, table64, w1_64, w2_64, w3_64;  // fp64 copies (NX_PRECISION_F64 scenes only)
    uint64_t version = next_scene_version();  // new on every change of parameters or settings
    nx_field_desc field{};
    nx_settings st{};
    int bad_status = NX_OK;
    std::string bad_msg;
    uint64_t validated_version = 0;  // the version bad_status describes
};

struct nx_frame {
    nx_ctx* ctx = nullptr;
    int device = 0;  // the creating context's device
    int W = 0, H = 0, K = 0, tiles_x = 0, tiles_y = 0;  // reference tiles (settings.tile)
    int list_tile = kWorkTile, ltiles_x = 0, ltiles_y = 0;  // tiles of the last built lists
    DevBuf base, ids, depths, weights, texture, final_img, residual;
    DevBuf base64;               // fp64 base kept for render_backward
    DevBuf residual64;           // fp64 terminal transmittance, kept with base64
    DevBuf tex_f;                // texture features (split tensor-core texture pass)
    DevBuf texture64, final64;   // fp64 texture / final (NX_PRECISION_F64 renders)
    bool f64 = false;            // the last collection pass rendered an NX_PRECISION_F64 scene
    bool keep_backward = false;  // collection passes write base64
    bool base64_valid = false;   // base64 holds the last forward's (or an uploaded) base
    DevBuf tile_offsets;  // n_tiles + 1 (the work lists' ranges of the last collection pass)
    DevBuf list_ids;
    uint64_t lists_gen = 0;  // the ctx's list build these lists came from (0: none)
    FrameStatsD* stats = nullptr;  // device
    int64_t n_nexels = 0;
    cudaEvent_t ev_ready = nullptr;  // collection pass of this frame done
    cudaEvent_t ev_busy = nullptr;   // last texture pass / download of this frame done
    bool busy_pending = false;
    // asynchronous list build: the device key count comes back in h_counts (ev_counts);
    // if it exceeded the capacity the build used, the frame is re-rendered from the
    // scene / camera it was rendered from before anything reads it
    int32_t* h_counts = nullptr;  // pinned [n_sorted, n_keys]
    cudaEvent_t ev_counts = nullptr;
    bool counts_pending = false;
    int64_t key_cap_used = 0;
    nx_camera cam{};
    const nx_scene* src_scene = nullptr;
    uint64_t src_version = 0;
    bool textured = false;
};

namespace {
// Scenes alive (a frame re-renders from its scene only if it still exists, unchanged).
std::mutex g_scenes_mu;
std::unordered_set<const nx_scene*> g_scenes;
void scene_alive(const nx_scene* s, bool alive) {
    std::lock_guard<std::mutex> lock(g_scenes_mu);
    if (alive) g_scenes.insert(s);
    else g_scenes.erase(s);
}
bool scene_is_alive(const nx_scene* s) {
    std::lock_guard<std::mutex> lock(g_scenes_mu);
    return g_scenes.count(s) > 0;
}
}  // namespace

namespace {

int set_err(nx_ctx* c, int status, const std::string& msg) {
    if (c) {
        c->err_status = status;
        c->err = msg;
    }
    return status;
}

int cuda_err(nx_ctx* c, cudaError_t e, const char* what) {
    return set_err(c, NX_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define NX_CUDA(ctx, expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return cuda_err(ctx, _e, #expr); \
    } while (0)

cudaStream_t pick_stream(nx_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

// validate_settings (renderer.cpp:13-21)
int validate_settings(nx_ctx* c, const nx_settings& s) {
    if (s.top_k < 0 || s.top_k > NX_MAX_TOP_K)
        return set_err(c, NX_BAD_SETTINGS, "top_k must be in [0, 8], got " + std::to_string(s.top_k));
    if (!(s.near_eps > 0)) return set_err(c, NX_BAD_SETTINGS, "near_eps must be positive");
    if (!(s.alpha_max > 0) || s.alpha_max >= 1) return set_err(c, NX_BAD_SETTINGS, "alpha_max must be in (0,1)");
    if (!(s.min_transmittance >= 0)) return set_err(c, NX_BAD_SETTINGS, "min_transmittance must be >= 0");
    if (s.tile < 1) return set_err(c, NX_BAD_SETTINGS, "tile must be >= 1");
    if (s.precision != NX_PRECISION_DEFAULT && s.precision != NX_PRECISION_F64)
        return set_err(c, NX_BAD_SETTINGS, "precision must be NX_PRECISION_DEFAULT or NX_PRECISION_F64");
    return NX_OK;
}

// validate_camera (camera.cpp:8-31)
int validate_camera(nx_ctx* c, const nx_camera& cam) {
    auto bad = [&](const char* what) { return set_err(c, NX_BAD_CAMERA, std::string("camera: ") + what); };
    if (cam.width <= 0 || cam.height <= 0) return bad("non-positive image size");
    if (!(cam.fx > 0) || !(cam.fy > 0)) return bad("non-positive focal length");
    for (int i = 0; i < 3; ++i) {
        if (!std::isfinite(cam.t[i])) return bad("non-finite translation");
        for (int j = 0; j < 3; ++j)
            if (!std::isfinite(cam.R[i * 3 + j])) return bad("non-finite rotation");
    }
    if (!std::isfinite(cam.cx) || !std::isfinite(cam.cy)) return bad("non-finite principal point");
    const double* R = cam.R;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double want = i == j ? 1.0 : 0.0;
            const double got = R[i * 3] * R[j * 3] + R[i * 3 + 1] * R[j * 3 + 1] + R[i * 3 + 2] * R[j * 3 + 2];
            if (std::abs(got - want) > 1e-9) return bad("rotation is not orthonormal");
        }
    const double cx = R[1] * R[5] - R[2] * R[4], cy = R[2] * R[3] - R[0] * R[5], cz = R[0] * R[4] - R[1] * R[3];
    if (cx * R[6] + cy * R[7] + cz * R[8] < 0) return bad("rotation is left-handed");
    return NX_OK;
}

CamD make_cam(const nx_camera& c) {
    CamD d;
    d.W = c.width;
    d.H = c.height;
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    for (int k = 0; k < 9; ++k) d.R[k] = c.R[k];
    for (int k = 0; k < 3; ++k) d.t[k] = c.t[k];
    // position() = -mul_transposed(R, t) (camera.hpp:24, vec_math.hpp:65-67)
    for (int k = 0; k < 3; ++k) d.o[k] = -(c.R[k] * c.t[0] + c.R[3 + k] * c.t[1] + c.R[6 + k] * c.t[2]);
    return d;
}

// Smallest cosine between a pixel-centre ray and the optical axis (at a corner pixel).
double min_axis_cosine(const nx_camera& c) {
    const double ax = std::max(std::abs((0.5 - c.cx) / c.fx), std::abs((c.width - 0.5 - c.cx) / c.fx));
    const double ay = std::max(std::abs((0.5 - c.cy) / c.fy), std::abs((c.height - 0.5 - c.cy) / c.fy));
    return 1.0 / std::sqrt(ax * ax + ay * ay + 1.0);
}

int bits_for(int64_t v) {
    int b = 0;
    while (b < 63 && (int64_t(1) << b) < v) ++b;
    return b;
}

int frame_shape(nx_ctx* c, nx_frame* f, int W, int H, int K, int tile) {
    const int64_t npix = static_cast<int64_t>(W) * H;
    NX_CUDA(c, f->base.ensure(npix * 3 * sizeof(float)));
    NX_CUDA(c, f->final_img.ensure(npix * 3 * sizeof(float)));
    NX_CUDA(c, f->residual.ensure(npix * sizeof(float)));
    const int64_t ns = std::max<int64_t>(npix * K, 1);
    NX_CUDA(c, f->ids.ensure(ns * sizeof(int32_t)));
    NX_CUDA(c, f->depths.ensure(ns * sizeof(double)));
    NX_CUDA(c, f->weights.ensure(ns * sizeof(double)));
    NX_CUDA(c, f->texture.ensure(ns * 3 * sizeof(float)));
    if (f->keep_backward || f->f64) {
        NX_CUDA(c, f->base64.ensure(npix * 3 * sizeof(double)));
        NX_CUDA(c, f->residual64.ensure(npix * sizeof(double)));
    }
    if (f->f64) {
        NX_CUDA(c, f->texture64.ensure(ns * 3 * sizeof(double)));
        NX_CUDA(c, f->final64.ensure(npix * 3 * sizeof(double)));
    }
    f->W = W;
    f->H = H;
    f->K = K;
    f->tiles_x = (W + tile - 1) / tile;
    f->tiles_y = (H + tile - 1) / tile;
    return NX_OK;
}

FrameDev frame_dev(const nx_frame* f) {
    FrameDev d;
    d.W = f->W;
    d.H = f->H;
    d.K = f->K;
    d.tiles_x = f->ltiles_x;  // the composite walks the lists of the last build (work tiles)
    d.tiles_y = f->ltiles_y;
    d.base = f->base.as<float>();
    d.ids = f->ids.as<int32_t>();
    d.depths = f->depths.as<double>();
    d.weights = f->weights.as<double>();
    d.texture = f->texture.as<float>();
    d.final_img = f->final_img.as<float>();
    d.residual = f->residual.as<float>();
    d.base64 = (f->keep_backward || f->f64) ? f->base64.as<double>() : nullptr;
    d.residual64 = (f->keep_backward || f->f64) ? f->residual64.as<double>() : nullptr;
    d.texture64 = f->f64 ? f->texture64.as<double>() : nullptr;
    d.final64 = f->f64 ? f->final64.as<double>() : nullptr;
    return d;
}

SceneDev scene_dev(const nx_scene* s) {
    SceneDev d;
    d.n = s->n;
    d.geom = s->geom.as<double>();
    d.sh = s->sh.as<float>();
    d.table = s->table.as<float>();
    d.w1 = s->w1.as<float>();
    d.w2 = s->w2.as<float>();
    d.w3 = s->w3.as<float>();
    d.field = s->field;
    const bool f64 = s->st.precision == NX_PRECISION_F64 && s->sh64.p;
    d.sh64 = f64 ? s->sh64.as<double>() : nullptr;
    d.table64 = f64 ? s->table64.as<double>() : nullptr;
    d.w1_64 = f64 ? s->w1_64.as<double>() : nullptr;
    d.w2_64 = f64 ? s->w2_64.as<double>() : nullptr;
    d.w3_64 = f64 ? s->w3_64.as<double>() : nullptr;
    return d;
}

void record(nx_ctx* c, int point, cudaStream_t s) {
    if (c->profiling) cudaEventRecord(c->ev[c->ev_cur][point], s);
}

// Folds a profiled frame's stage events into the running sums. Non-blocking unless
// `wait`: a set whose last event has not completed yet stays pending.
void fold_set(nx_ctx* c, int set, bool wait) {
    if (!c->ev_pending[set]) return;
    cudaEvent_t last = c->ev[set][kEvTexEnd];
    if (wait) cudaEventSynchronize(last);
    else if (cudaEventQuery(last) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    static const int kFrom[NX_NUM_STAGES] = {kEvPre, kEvDepth, kEvEmit, kEvTileSort, kEvComp, kEvTex, kEvTexMid};
    static const int kTo[NX_NUM_STAGES] = {kEvDepth, kEvEmit, kEvTileSort, kEvComp, kEvCompEnd, kEvTexEnd, kEvTexEnd};
    for (int i = 0; i < NX_NUM_STAGES; ++i) {
        float v = 0.f;
        if (cudaEventElapsedTime(&v, c->ev[set][kFrom[i]], c->ev[set][kTo[i]]) == cudaSuccess) c->stage_acc[i] += v;
    }
    cudaGetLastError();
    c->stage_frames += 1;
    c->ev_pending[set] = false;
}

// Called at the start of each profiled frame: folds whatever completed and moves to
// the next event set of the ring (blocking only if that set is still in flight).
void next_event_set(nx_ctx* c) {
    for (int s = 0; s < kEvSets; ++s) fold_set(c, s, false);
    c->ev_cur = (c->ev_cur + 1) % kEvSets;
    fold_set(c, c->ev_cur, true);
}

const char* const kBadWhat[] = {"non-finite position", "non-finite quaternion", "non-finite log scale",
                                "non-finite kernel exponent", "non-finite opacity", "non-finite sh coefficient",
                                "degenerate quaternion"};

// The reference activates every primitive on every render (renderer.cpp:38,
// primitive.cpp:47-63). Scenes are validated when created; after any change of their
// parameters (Adam, set_params, densify, prune: a new version) the next render
// re-runs the checks on the device before using them (one small read-back).
int revalidate(nx_ctx* c, nx_scene* scene, cudaStream_t s) {
    if (scene->validated_version == scene->version) return NX_OK;
    NX_CUDA(c, c->valid_word.ensure(sizeof(unsigned long long)));
    unsigned long long* first = c->valid_word.as<unsigned long long>();
    NX_CUDA(c, cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), s));
    launch_validate(scene->geom.as<double>(), scene->sh.as<float>(), scene->n, first, s);
    unsigned long long* h = reinterpret_cast<unsigned long long*>(c->h_pinned + 32);
    NX_CUDA(c, cudaMemcpyAsync(h, first, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    const unsigned long long v = *h;
    if (v == ~0ull) {
        scene->bad_status = NX_OK;
        scene->bad_msg.clear();
    } else {
        scene->bad_status = NX_BAD_PRIMITIVE;
        scene->bad_msg = std::string(kBadWhat[v & 7]) + " in primitive " + std::to_string(v >> 3);
    }
    scene->validated_version = scene->version;
    return NX_OK;
}

int check_inputs(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, cudaStream_t s = nullptr) {
    if (!c || !scene || !cam) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    int st;
    if ((st = validate_settings(c, scene->st))) return st;
    if ((st = validate_camera(c, *cam))) return st;
    // on the caller's stream, after whatever changed the parameters there
    if ((st = revalidate(c, const_cast<nx_scene*>(scene), s ? s : c->stream))) return st;
    if (scene->bad_status) return set_err(c, scene->bad_status, scene->bad_msg);
    return NX_OK;
}

// Builds the per-tile lists (work lists, or the reference lists when
// reference_lists) for `cam` into frame->list_ids / frame->tile_offsets.
int build_lists(nx_ctx* c, const nx_scene* scene, const nx_camera& cam, nx_frame* f, int reference_lists,
                cudaStream_t s, int64_t* total_keys, int work_tile = kWorkTile, bool allow_async = false) {
    const int64_t n = scene->n;
    // list geometry: reference lists per settings.tile, work lists per work_tile
    const int lt = reference_lists ? scene->st.tile : work_tile;
    f->list_tile = lt;
    f->ltiles_x = (cam.width + lt - 1) / lt;
    f->ltiles_y = (cam.height + lt - 1) / lt;
    const int64_t n_tiles = static_cast<int64_t>(f->ltiles_x) * f->ltiles_y;
    const CamD cd = make_cam(cam);
    const int64_t nn = std::max<int64_t>(n, 1);
    NX_CUDA(c, c->rec.ensure(nn * REC_FIELDS * sizeof(double)));
    NX_CUDA(c, c->recf.ensure(nn * 4 * sizeof(float4)));
    NX_CUDA(c, c->cls.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->ref_rect.ensure(nn * sizeof(int4)));
    NX_CUDA(c, c->work_rect.ensure(nn * sizeof(int4)));
    NX_CUDA(c, c->key.ensure(nn * sizeof(uint64_t)));
    NX_CUDA(c, c->flag.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->pos.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->skeys_a.ensure(nn * sizeof(uint64_t)));
    NX_CUDA(c, c->skeys_b.ensure(nn * sizeof(uint64_t)));
    NX_CUDA(c, c->sids_a.ensure(nn * sizeof(uint32_t)));
    NX_CUDA(c, c->sids_b.ensure(nn * sizeof(uint32_t)));
    NX_CUDA(c, c->counts.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->offsets.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->tile_counts.ensure((n_tiles + 1) * sizeof(int32_t)));
    NX_CUDA(c, f->tile_offsets.ensure((n_tiles + 1) * sizeof(int32_t)));
    const size_t scratch_ints =
        std::max({scan_scratch_ints(nn), radix_scratch_ints64(nn), scan_scratch_ints(n_tiles + 1)}) + 64;
    NX_CUDA(c, c->scratch.ensure(scratch_ints * sizeof(int32_t)));
    NX_CUDA(c, cudaMemsetAsync(f->stats, 0, sizeof(FrameStatsD), s));

    if (c->profiling) next_event_set(c);
    record(c, kEvPre, s);
    PreprocessArgs pa;
    pa.scene = scene_dev(scene);
    pa.st = scene->st;
    pa.cam = cd;
    pa.tiles_x = f->tiles_x;
    pa.tiles_y = f->tiles_y;
    pa.work_tile = lt;
    pa.zmin_work = 0.5 * scene->st.near_eps * min_axis_cosine(cam);
    pa.rec = c->rec.as<double>();
    pa.recf = c->recf.as<float4>();
    pa.cls = c->cls.as<int32_t>();
    pa.ref_rect = c->ref_rect.as<int4>();
    pa.work_rect = c->work_rect.as<int4>();
    pa.key = c->key.as<uint64_t>();
    pa.flag = c->flag.as<int32_t>();
    pa.reference_lists = reference_lists;
    pa.stats = f->stats;
    launch_preprocess(pa, s);

    // K2: compaction of the primitives that own work (id-ascending) + depth sort.
    int32_t* d_total = c->scratch.as<int32_t>();  // [0] n_sorted, [1] n_keys
    int32_t* sc = d_total + 64;
    // The sorted count stays on the device: the sort runs over capacity n with the
    // device count (no host round trip).
    scan_exclusive(c->flag.as<int32_t>(), c->pos.as<int32_t>(), n, d_total, sc, s);
    record(c, kEvDepth, s);
    launch_compact(c->flag.as<int32_t>(), c->pos.as<int32_t>(), c->key.as<uint64_t>(), n, c->skeys_a.as<uint64_t>(),
                   c->sids_a.as<uint32_t>(), s);
    const bool in_b = radix_sort_pairs_u64(c->skeys_a.as<uint64_t>(), c->sids_a.as<uint32_t>(),
                                           c->skeys_b.as<uint64_t>(), c->sids_b.as<uint32_t>(), n, d_total, 0, 64, sc,
                                           s);
    const uint32_t* sorted_ids = in_b ? c->sids_b.as<uint32_t>() : c->sids_a.as<uint32_t>();
    const uint64_t* sorted_keys = in_b ? c->skeys_b.as<uint64_t>() : c->skeys_a.as<uint64_t>();

    // K3: emit (tile, id) keys in sorted order. The key count stays on the device: the
    // keys go into buffers of the context's capacity (grow-only) and the count comes back
    // asynchronously (frame_settle re-renders a frame that exceeded it). Without a
    // capacity yet (first frame), for reference lists and for debug / backward builds,
    // the count is read back first (one host round trip) and sizes the buffers exactly.
    record(c, kEvEmit, s);
    launch_rect_counts(sorted_ids, n, d_total, c->work_rect.as<int4>(), c->counts.as<int32_t>(), sorted_keys, f->stats,
                       s);
    scan_exclusive(c->counts.as<int32_t>(), c->offsets.as<int32_t>(), n, d_total + 1, sc, s);
    const bool async = allow_async && !reference_lists && c->key_cap > 0 && !c->sync_lists && f->h_counts;
    int64_t cap;
    if (async) {
        cap = c->key_cap;
    } else {
        NX_CUDA(c, cudaMemcpyAsync(c->h_pinned, d_total, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        NX_CUDA(c, cudaStreamSynchronize(s));
        const int64_t n_sorted = n > 0 ? c->h_pinned[0] : 0;
        const int64_t n_keys = n_sorted > 0 ? c->h_pinned[1] : 0;
        if (n_keys < 0) return set_err(c, NX_UNSUPPORTED, "tile-key count exceeds 2^31");
        cap = std::max<int64_t>(n_keys, 1);
        if (!reference_lists) c->key_cap = std::max(c->key_cap, n_keys + n_keys / 4 + 4096);
        *total_keys = n_keys;
    }
    NX_CUDA(c, c->tkeys_a.ensure(cap * sizeof(uint32_t)));
    NX_CUDA(c, c->tkeys_b.ensure(cap * sizeof(uint32_t)));
    NX_CUDA(c, c->tvals_a.ensure(cap * sizeof(uint32_t)));
    NX_CUDA(c, c->tvals_b.ensure(cap * sizeof(uint32_t)));
    const size_t need = radix_scratch_ints(cap) + 64;
    if (need * sizeof(int32_t) > c->scratch.cap) {
        // grow the scratch, keeping the device totals
        DevBuf grown;
        NX_CUDA(c, grown.ensure(need * sizeof(int32_t)));
        NX_CUDA(c, cudaMemcpyAsync(grown.p, c->scratch.p, 64 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        NX_CUDA(c, cudaStreamSynchronize(s));
        std::swap(c->scratch.p, grown.p);
        std::swap(c->scratch.cap, grown.cap);
        grown.release();
        d_total = c->scratch.as<int32_t>();
        sc = d_total + 64;
    }
    NX_CUDA(c, cudaMemsetAsync(c->tile_counts.as<int32_t>(), 0, (n_tiles + 1) * sizeof(int32_t), s));
    EmitCull cull;  // work lists: keys the corner-ray quadrilateral proves empty go past the last tile
    cull.n_tiles = static_cast<int>(n_tiles);
    if (!reference_lists && c->emit_cull) {
        cull.recf = c->recf.as<float4>();
        cull.tiles_x = f->ltiles_x;
        cull.tile = lt;
        cull.W = cam.width;
        cull.H = cam.height;
        cull.cx = static_cast<float>(cd.cx);
        cull.cy = static_cast<float>(cd.cy);
        cull.ifx = static_cast<float>(1.0 / cd.fx);
        cull.ify = static_cast<float>(1.0 / cd.fy);
        for (int q = 0; q < 9; ++q) cull.R[q] = static_cast<float>(cd.R[q]);
    }
    launch_emit(sorted_ids, c->offsets.as<int32_t>(), n, d_total, cap, d_total + 1, c->work_rect.as<int4>(),
                f->ltiles_x, c->tkeys_a.as<uint32_t>(), c->tvals_a.as<uint32_t>(), c->tile_counts.as<int32_t>(), cull,
                s);

    // K4: stable sort by tile (over the device count, capped by the capacity); the cull's
    // sentinel n_tiles sorts past every list
    record(c, kEvTileSort, s);
    const int tb = std::max(bits_for(n_tiles + 1), 1);
    const bool t_in_b = radix_sort_pairs_u32(c->tkeys_a.as<uint32_t>(), c->tvals_a.as<uint32_t>(),
                                             c->tkeys_b.as<uint32_t>(), c->tvals_b.as<uint32_t>(), cap, d_total + 1,
                                             0, tb, sc, s);
    f->key_cap_used = cap;
    f->counts_pending = false;
    if (async) {
        *total_keys = -1;  // on the device; f->h_counts once ev_counts completes
        NX_CUDA(c, cudaMemcpyAsync(f->h_counts, d_total, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        NX_CUDA(c, cudaEventRecord(f->ev_counts, s));
        f->counts_pending = true;
    }
    // K5: tile ranges.
    scan_exclusive(c->tile_counts.as<int32_t>(), f->tile_offsets.as<int32_t>(), n_tiles + 1, nullptr, sc, s);
    f->list_ids.p = t_in_b ? c->tvals_b.p : c->tvals_a.p;  // borrowed (not owned)
    f->list_ids.cap = 0;
    c->lists_gen += 1;
    f->lists_gen = reference_lists ? 0 : c->lists_gen;
    c->lists_scene = scene;
    c->lists_scene_version = scene->version;
    c->lists_cam = cam;
    c->lists_tile = reference_lists ? 0 : lt;
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

int collection(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, cudaStream_t s,
               int32_t* dbg_hits, int32_t* dbg_counts, int dbg_y0, int dbg_y1, int dbg_max);
int texturing(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, cudaStream_t s);

// Before anything reads a frame back: if its list build ran on a capacity and the key
// count it reported exceeds it, the capacity grows and the frame is rendered again from
// the same scene (alive and unchanged) and camera, synchronously.
int frame_settle(nx_ctx* c, nx_frame* f) {
    if (!f->counts_pending) return NX_OK;
    NX_CUDA(c, cudaEventSynchronize(f->ev_counts));
    f->counts_pending = false;
    const int64_t n_keys = f->h_counts[0] > 0 ? f->h_counts[1] : 0;
    c->key_cap = std::max(c->key_cap, n_keys + n_keys / 4 + 4096);
    if (n_keys <= f->key_cap_used) return NX_OK;
    if (!f->src_scene || !scene_is_alive(f->src_scene) || f->src_scene->version != f->src_version)
        return set_err(c, NX_INVALID_ARGUMENT,
                       "frame exceeded the work-list capacity and its scene changed since: render it again");
    const nx_camera cam = f->cam;
    const bool tex = f->textured;
    int st = collection(c, f->src_scene, &cam, f, c->stream, nullptr, nullptr, 0, 0, 0);
    if (!st && tex) st = texturing(c, f->src_scene, &cam, f, c->stream);
    if (st) return st;
    NX_CUDA(c, cudaStreamSynchronize(c->stream));
    return f->counts_pending ? frame_settle(c, f) : NX_OK;
}

int collection(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, cudaStream_t s,
               int32_t* dbg_hits, int32_t* dbg_counts, int dbg_y0, int dbg_y1, int dbg_max) {
    int st;
    if ((st = check_inputs(c, scene, cam, s))) return st;
    // the frame may still be read by its previous texture pass / download (second stream)
    if (f->busy_pending) NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_busy, 0));
    f->f64 = scene->st.precision == NX_PRECISION_F64;
    if ((st = frame_shape(c, f, cam->width, cam->height, scene->st.top_k, scene->st.tile))) return st;
    f->n_nexels = scene->n;
    int64_t total = 0;
    f->cam = *cam;
    f->src_scene = scene;
    f->src_version = scene->version;
    f->textured = false;
    if ((st = build_lists(c, scene, *cam, f, 0, s, &total, kWorkTile, dbg_hits == nullptr))) return st;
    record(c, kEvComp, s);
    CompositeArgs ca;
    ca.rec = c->rec.as<double>();
    ca.recf = c->recf.as<float4>();
    ca.n = std::max<int64_t>(scene->n, 1);
    ca.sh = scene->sh.as<float>();
    ca.list_ids = f->list_ids.as<int32_t>();
    ca.tile_offsets = f->tile_offsets.as<int32_t>();
    ca.st = scene->st;
    ca.cam = make_cam(*cam);
    ca.fb = frame_dev(f);
    ca.sh_degree = scene->st.no_prim_sh ? 0 : 3;
    ca.dbg_hits = dbg_hits;
    ca.dbg_counts = dbg_counts;
    ca.dbg_y0 = dbg_y0;
    ca.dbg_y1 = dbg_y1;
    ca.dbg_max = dbg_max;
    ca.stats = f->stats;
    ca.sh64 = scene_dev(scene).sh64;
    // frames that keep the backward state (training) and fp64-colour frames composite on
    // the exact fp64 path; display frames on the certified fp32 alpha + exact redo
    ca.certified = c->certified && !f->keep_backward && !f->f64;
    if (ca.certified) {
        NX_CUDA(c, c->redo.ensure((static_cast<int64_t>(cam->width) * cam->height + 1) * sizeof(int32_t)));
        NX_CUDA(c, cudaMemsetAsync(c->redo.p, 0, sizeof(int32_t), s));
        ca.redo = c->redo.as<int32_t>();
        ca.redo_all = c->redo_all;
    }
    launch_composite(ca, s);
    f->base64_valid = f->keep_backward || f->f64;
    record(c, kEvCompEnd, s);
    NX_CUDA(c, cudaEventRecord(f->ev_ready, s));
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

int texturing(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, cudaStream_t s) {
    if (f->W != cam->width || f->H != cam->height)
        return set_err(c, NX_INVALID_ARGUMENT, "frame does not match the camera (run collection_pass first)");
    NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_ready, 0));  // no-op on the collection's own stream
    if (scene->st.precision == NX_PRECISION_F64 && !f->f64) {  // e.g. a frame uploaded from host buffers
        if (!f->base64_valid)
            return set_err(c, NX_INVALID_ARGUMENT, "NX_PRECISION_F64 texturing needs the frame's fp64 base");
        f->f64 = true;
        if (const int st = frame_shape(c, f, f->W, f->H, f->K, scene->st.tile)) return st;
    }
    record(c, kEvTex, s);
    TextureArgs ta;
    ta.scene = scene_dev(scene);
    ta.st = scene->st;
    ta.cam = make_cam(*cam);
    ta.fb = frame_dev(f);
    ta.stats = f->stats;
    ta.fscratch = nullptr;
    ta.ev_mid = c->profiling ? c->ev[c->ev_cur][kEvTexMid] : nullptr;  // recorded between gathers and decoder
    if (texture_tc_supported(scene->st.top_k > 0 ? scene->field : nx_field_desc{}) && f->K > 0 && !f->f64) {
        const size_t bytes = texture_tc_scratch_bytes(f->W, f->H, f->K);
        if (bytes) {
            if (bytes > f->tex_f.cap) {  // zeroed once: padding rows of the tiles are never written
                NX_CUDA(c, f->tex_f.ensure(bytes));
                NX_CUDA(c, cudaMemsetAsync(f->tex_f.p, 0, f->tex_f.cap, s));
            }
            ta.fscratch = f->tex_f.as<float>();
        }
    }
    const int st = launch_texture(ta, s);
    if (st) return set_err(c, st, "texture field shape not supported (n_in <= 64, n_hidden <= 128)");
    if (c->profiling && !ta.ev_mid_recorded) record(c, kEvTexMid, s);  // no separate decoder launch
    record(c, kEvTexEnd, s);
    if (c->profiling) c->ev_pending[c->ev_cur] = true;
    NX_CUDA(c, cudaEventRecord(f->ev_busy, s));
    f->busy_pending = true;
    f->textured = true;
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

}  // namespace

extern "C" {

uint64_t nx_launch_count(void) { return g_launches.load(); }

const char* nx_version(void) { return "nexel-b200 0.1 (sm_100a)"; }

const char* nx_status_name(int status) {
    switch (status) {
        case NX_OK: return "ok";
        case NX_BAD_SETTINGS: return "bad-settings";
        case NX_BAD_CAMERA: return "bad-camera";
        case NX_BAD_PRIMITIVE: return "bad-primitive";
        case NX_MISSING_FILE: return "missing-file";
        case NX_BAD_CHECKPOINT: return "bad-checkpoint";
        case NX_INVALID_ARGUMENT: return "invalid-argument";
        case NX_UNSUPPORTED: return "unsupported";
        case NX_OUT_OF_MEMORY: return "out-of-memory";
        case NX_CUDA_ERROR: return "cuda-error";
        case NX_NO_DEVICE: return "no-device";
        default: return "unknown";
    }
}

const char* nx_stage_name(int stage) { return stage >= 0 && stage < NX_NUM_STAGES ? kStageNames[stage] : "?"; }

int nx_device_count(int* count) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    *count = e == cudaSuccess ? n : 0;
    return e == cudaSuccess ? NX_OK : NX_NO_DEVICE;
}

int nx_ctx_create(int device, nx_ctx** out) {
    if (!out) return NX_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return NX_NO_DEVICE;
    if (cudaSetDevice(device) != cudaSuccess) return NX_NO_DEVICE;
    nx_ctx* c = new (std::nothrow) nx_ctx;
    if (!c) return NX_OUT_OF_MEMORY;
    c->device = device;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (const char* e = std::getenv("NX_SYNC_LISTS")) c->sync_lists = std::atoi(e) != 0;
    if (const char* e = std::getenv("NX_CERTIFIED")) c->certified = std::atoi(e) != 0;
    if (const char* e = std::getenv("NX_EMIT_CULL")) c->emit_cull = std::atoi(e) != 0;
    if (const char* e = std::getenv("NX_CERT_REDO_ALL")) c->redo_all = std::atoi(e) != 0;
    if (const char* e = std::getenv("NX_KEY_CAP")) c->key_cap = std::atoll(e);  // tests: start from a small capacity
    // The collection stream outranks the texture stream: the block scheduler hands the next
    // frame's latency-bound binning kernels SMs ahead of the remaining CTAs of the
    // previous frame's texture gathers, which fill the gaps instead of blocking them
    // (NX_STREAM_PRIORITY=0: equal priorities).
    int prio_low = 0, prio_high = 0;
    cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    if (const char* e = std::getenv("NX_STREAM_PRIORITY"))
        if (std::atoi(e) == 0) prio_low = prio_high = 0;
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_high) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_low) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream3, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream_bwd, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_bwd_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_bwd_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaMallocHost(&c->h_pinned, 64 * sizeof(int32_t)) != cudaSuccess) {
        delete c;
        return NX_CUDA_ERROR;
    }
    for (auto& set : c->ev)
        for (auto& e : set) cudaEventCreate(&e);
    *out = c;
    return NX_OK;
}

void nx_ctx_destroy(nx_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->stream2);
    cudaStreamSynchronize(c->stream3);
    cudaStreamSynchronize(c->stream_bwd);
    for (DevBuf* b : {&c->rec, &c->recf, &c->cls, &c->ref_rect, &c->work_rect, &c->key, &c->flag, &c->pos, &c->skeys_a,
                      &c->skeys_b, &c->sids_a, &c->sids_b, &c->counts, &c->offsets, &c->tkeys_a, &c->tkeys_b,
                      &c->tvals_a, &c->tvals_b, &c->tile_counts, &c->scratch, &c->dbg_hits, &c->dbg_counts, &c->valid_word})
        b->release();
    for (DevBuf* b : {&c->d_t_slot, &c->act_grad, &c->xacc_prims, &c->dens_map, &c->dens_par, &c->dens_src, &c->h_err, &c->h_blend, &c->loss_scratch, &c->h_gt, &c->h_terms})
        b->release();
    c->field_bwd.release();
    for (DevBuf& b : c->h_up) b.release();
    for (DevBuf& b : c->h_grads) b.release();
    if (c->bwd_lists) nx_frame_destroy(c->bwd_lists);
    for (auto& set : c->ev)
        for (auto& e : set) cudaEventDestroy(e);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    cudaEventDestroy(c->ev_join);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->stream2);
    cudaStreamDestroy(c->stream3);
    cudaEventDestroy(c->ev_bwd_fork);
    cudaEventDestroy(c->ev_bwd_join);
    cudaStreamDestroy(c->stream_bwd);
    delete c;
}

const char* nx_ctx_last_error(const nx_ctx* c, int* status) {
    if (!c) return "null context";
    if (status) *status = c->err_status;
    return c->err.c_str();
}

void* nx_ctx_stream(nx_ctx* c) { return c ? c->stream : nullptr; }

int nx_ctx_synchronize(nx_ctx* c) {
    NX_CUDA(c, cudaStreamSynchronize(c->stream));
    NX_CUDA(c, cudaStreamSynchronize(c->stream2));
    NX_CUDA(c, cudaStreamSynchronize(c->stream3));
    return NX_OK;
}

int nx_ctx_join(nx_ctx* c) {
    if (!c) return NX_INVALID_ARGUMENT;
    for (cudaStream_t s2 : {c->stream2, c->stream3}) {
        NX_CUDA(c, cudaEventRecord(c->ev_join, s2));
        NX_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
    return NX_OK;
}

int nx_ctx_set_profiling(nx_ctx* c, int enable) {
    if (!c) return NX_INVALID_ARGUMENT;
    c->profiling = enable != 0;
    return NX_OK;
}

int nx_ctx_stage_times(nx_ctx* c, float* ms, int n, int* frames) {
    if (!c || !ms) return NX_INVALID_ARGUMENT;
    NX_CUDA(c, cudaDeviceSynchronize());
    for (int set = 0; set < kEvSets; ++set) fold_set(c, set, true);
    for (int i = 0; i < n && i < NX_NUM_STAGES; ++i)
        ms[i] = c->stage_frames ? static_cast<float>(c->stage_acc[i] / c->stage_frames) : 0.f;
    if (frames) *frames = c->stage_frames;
    for (double& v : c->stage_acc) v = 0.0;
    c->stage_frames = 0;
    return NX_OK;
}

int nx_scene_create(nx_ctx* c, const nx_settings* settings, int64_t n, const double* nexels,
                    const nx_field_desc* field, const double* table, const double* w1, const double* w2,
                    const double* w3, nx_scene** out) {
    if (!c || !settings || !field || !out || n < 0 || (n > 0 && !nexels) || !table || !w1 || !w2 || !w3)
        return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (n >= (int64_t(1) << 31)) return set_err(c, NX_UNSUPPORTED, "more than 2^31 primitives");
    if (field->levels < 1 || field->features < 1 || field->n_hidden < 1 || field->log2_table < 0 ||
        field->log2_table > 30)
        return set_err(c, NX_INVALID_ARGUMENT, "bad field description");
    cudaSetDevice(c->device);
    nx_scene* s = new (std::nothrow) nx_scene;
    if (!s) return set_err(c, NX_OUT_OF_MEMORY, "host allocation");
    s->ctx = c;
    s->device = c->device;
    s->n = n;
    s->field = *field;
    s->st = *settings;
    // Validation exactly as activate() (primitive.cpp:47-63), first failing id.
    const char* const* whats = kBadWhat;
    for (int64_t i = 0; i < n && !s->bad_status; ++i) {
        const double* p = nexels + i * NX_PARAMS_PER_NEXEL;
        int what = -1;
        for (int k = 0; k < 3 && what < 0; ++k)
            if (!std::isfinite(p[k])) what = 0;
        for (int k = 0; k < 4 && what < 0; ++k)
            if (!std::isfinite(p[3 + k])) what = 1;
        for (int k = 0; k < 2 && what < 0; ++k) {
            if (!std::isfinite(p[7 + k])) what = 2;
            else if (!std::isfinite(p[10 + k])) what = 3;
        }
        if (what < 0 && !std::isfinite(p[9])) what = 4;
        for (int k = 0; k < NX_SH_VALUES && what < 0; ++k)
            if (!std::isfinite(p[12 + k])) what = 5;
        if (what < 0) {
            const double qn = std::sqrt(p[3] * p[3] + p[4] * p[4] + p[5] * p[5] + p[6] * p[6]);
            if (!(qn > 1e-12)) what = 6;
        }
        if (what >= 0) {
            s->bad_status = NX_BAD_PRIMITIVE;
            s->bad_msg = std::string(whats[what]) + " in primitive " + std::to_string(i);
        }
    }
    const int64_t nn = std::max<int64_t>(n, 1);
    std::vector<double> geom(static_cast<size_t>(kGeomFields * nn), 0.0);
    std::vector<float> sh(static_cast<size_t>(NX_SH_VALUES * nn), 0.f);
    for (int64_t i = 0; i < n; ++i) {
        const double* p = nexels + i * NX_PARAMS_PER_NEXEL;
        for (int k = 0; k < kGeomFields; ++k) geom[k * nn + i] = p[k];
        for (int k = 0; k < NX_SH_VALUES; ++k) sh[i * NX_SH_VALUES + k] = static_cast<float>(p[12 + k]);
    }
    const size_t n_table = static_cast<size_t>(field->levels) * (size_t(1) << field->log2_table) * field->features;
    const size_t n_in = static_cast<size_t>(field->levels) * field->features;
    const size_t nh = field->n_hidden;
    auto upload_f32 = [&](DevBuf& b, const double* src, size_t count) -> cudaError_t {
        cudaError_t e = b.ensure(std::max<size_t>(count, 1) * sizeof(float));
        if (e != cudaSuccess) return e;
        std::vector<float> tmp(std::min<size_t>(count, size_t(1) << 22));
        for (size_t at = 0; at < count; at += tmp.size()) {
            const size_t m = std::min(tmp.size(), count - at);
            for (size_t k = 0; k < m; ++k) tmp[k] = static_cast<float>(src[at + k]);
            e = cudaMemcpy(b.as<float>() + at, tmp.data(), m * sizeof(float), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    };
    cudaError_t e = s->geom.ensure(geom.size() * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(s->geom.p, geom.data(), geom.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = s->sh.ensure(sh.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(s->sh.p, sh.data(), sh.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = upload_f32(s->table, table, n_table);
    if (e == cudaSuccess) e = upload_f32(s->w1, w1, nh * n_in);
    if (e == cudaSuccess) e = upload_f32(s->w2, w2, nh * nh);
    if (e == cudaSuccess) e = upload_f32(s->w3, w3, NX_SH_VALUES * nh);
    if (settings->precision == NX_PRECISION_F64) {  // fp64 copies of everything the colour path reads
        std::vector<double> sh64(static_cast<size_t>(NX_SH_VALUES * nn), 0.0);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < NX_SH_VALUES; ++k) sh64[i * NX_SH_VALUES + k] = nexels[i * NX_PARAMS_PER_NEXEL + 12 + k];
        auto up64 = [&](DevBuf& b, const double* src, size_t count) -> cudaError_t {
            cudaError_t e2 = b.ensure(std::max<size_t>(count, 1) * sizeof(double));
            if (e2 == cudaSuccess && count) e2 = cudaMemcpy(b.p, src, count * sizeof(double), cudaMemcpyHostToDevice);
            return e2;
        };
        if (e == cudaSuccess) e = up64(s->sh64, sh64.data(), sh64.size());
        if (e == cudaSuccess) e = up64(s->table64, table, n_table);
        if (e == cudaSuccess) e = up64(s->w1_64, w1, nh * n_in);
        if (e == cudaSuccess) e = up64(s->w2_64, w2, nh * nh);
        if (e == cudaSuccess) e = up64(s->w3_64, w3, NX_SH_VALUES * nh);
    }
    // pageable cudaMemcpy may return before its DMA lands, and the context's
    // non-blocking streams do not order after the legacy stream: finish it here
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        nx_scene_destroy(s);
        return cuda_err(c, e, "scene upload");
    }
    s->validated_version = s->version;  // validated above, on the host
    scene_alive(s, true);
    *out = s;
    return NX_OK;
}

// load_checkpoint (checkpoint.cpp:173-271) into a device scene. The parameter
// sections are fp32 SoA on disk; positions / shape parameters become the fp64
// geometry rows (exact widening), SH, table and MLP weights are uploaded as stored.
int nx_scene_load_nexl(nx_ctx* c, const char* path, nx_scene** out, nx_nexl_info* info) {
    if (!c || !path || !out) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    NexlHeader h;
    NexlArrays arr;
    std::string err;
    int st = nexl_read(path, true, h, &arr, err);
    if (st) return set_err(c, st, err);
    if (h.info.n_nexels >= (int64_t(1) << 31)) return set_err(c, NX_UNSUPPORTED, "more than 2^31 primitives");
    cudaSetDevice(c->device);
    nx_scene* s = new (std::nothrow) nx_scene;
    if (!s) return set_err(c, NX_OUT_OF_MEMORY, "host allocation");
    s->ctx = c;
    s->device = c->device;
    const int64_t n = h.info.n_nexels;
    s->n = n;
    s->field = h.info.field;
    s->st = h.info.settings;
    // validation exactly as activate() (primitive.cpp:47-63), first failing id
    const char* const* whats = kBadWhat;
    for (int64_t i = 0; i < n && !s->bad_status; ++i) {
        int what = -1;
        for (int k = 0; k < 3 && what < 0; ++k)
            if (!std::isfinite(arr.mu[i * 3 + k])) what = 0;
        for (int k = 0; k < 4 && what < 0; ++k)
            if (!std::isfinite(arr.quat[i * 4 + k])) what = 1;
        for (int k = 0; k < 2 && what < 0; ++k) {
            if (!std::isfinite(arr.log_scale[i * 2 + k])) what = 2;
            else if (!std::isfinite(arr.gamma[i * 2 + k])) what = 3;
        }
        if (what < 0 && !std::isfinite(arr.opacity[i])) what = 4;
        for (int k = 0; k < NX_SH_VALUES && what < 0; ++k)
            if (!std::isfinite(arr.sh[i * NX_SH_VALUES + k])) what = 5;
        if (what < 0) {
            double qn = 0.0;
            for (int k = 0; k < 4; ++k) qn += static_cast<double>(arr.quat[i * 4 + k]) * arr.quat[i * 4 + k];
            if (!(std::sqrt(qn) > 1e-12)) what = 6;
        }
        if (what >= 0) {
            s->bad_status = NX_BAD_PRIMITIVE;
            s->bad_msg = std::string(whats[what]) + " in primitive " + std::to_string(i);
        }
    }
    const int64_t nn = std::max<int64_t>(n, 1);
    std::vector<double> geom(static_cast<size_t>(kGeomFields * nn), 0.0);
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) geom[k * nn + i] = arr.mu[i * 3 + k];
        for (int k = 0; k < 4; ++k) geom[(3 + k) * nn + i] = arr.quat[i * 4 + k];
        for (int k = 0; k < 2; ++k) geom[(7 + k) * nn + i] = arr.log_scale[i * 2 + k];
        geom[9 * nn + i] = arr.opacity[i];
        for (int k = 0; k < 2; ++k) geom[(10 + k) * nn + i] = arr.gamma[i * 2 + k];
    }
    auto up = [&](DevBuf& b, const void* src, size_t bytes) -> cudaError_t {
        cudaError_t e = b.ensure(std::max<size_t>(bytes, 4));
        if (e == cudaSuccess && bytes) e = cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    cudaError_t e = up(s->geom, geom.data(), geom.size() * sizeof(double));
    if (e == cudaSuccess) e = up(s->sh, arr.sh.data(), arr.sh.size() * sizeof(float));
    if (e == cudaSuccess) e = up(s->table, arr.table.data(), arr.table.size() * sizeof(float));
    if (e == cudaSuccess) e = up(s->w1, arr.w1.data(), arr.w1.size() * sizeof(float));
    if (e == cudaSuccess) e = up(s->w2, arr.w2.data(), arr.w2.size() * sizeof(float));
    if (e == cudaSuccess) e = up(s->w3, arr.w3.data(), arr.w3.size() * sizeof(float));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // pageable copies complete before stream work
    if (e != cudaSuccess) {
        nx_scene_destroy(s);
        return cuda_err(c, e, "checkpoint upload");
    }
    if (info) *info = h.info;
    s->validated_version = s->version;  // validated above, on the host
    scene_alive(s, true);
    *out = s;
    return NX_OK;
}

int nx_scene_set_settings(nx_ctx* c, nx_scene* s, const nx_settings* settings) {
    if (!s || !settings) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (settings->precision == NX_PRECISION_F64 && !s->sh64.p)
        return set_err(c, NX_UNSUPPORTED, "NX_PRECISION_F64 needs a scene created with it (fp64 copies)");
    if (std::memcmp(&s->st, settings, sizeof(nx_settings)) != 0) s->version = next_scene_version();
    s->st = *settings;
    return NX_OK;
}

int nx_scene_get_settings(const nx_scene* s, nx_settings* out) {
    if (!s || !out) return NX_INVALID_ARGUMENT;
    *out = s->st;
    return NX_OK;
}

void nx_scene_destroy(nx_scene* s) {
    if (!s) return;
    scene_alive(s, false);
    cudaSetDevice(s->device);
    for (DevBuf* b : {&s->geom, &s->sh, &s->table, &s->w1, &s->w2, &s->w3, &s->geom_spare, &s->sh_spare, &s->sh64,
                      &s->table64, &s->w1_64, &s->w2_64, &s->w3_64})
        b->release();
    delete s;
}

int nx_frame_create(nx_ctx* c, int width, int height, int top_k, nx_frame** out) {
    if (!c || !out || width < 0 || height < 0 || top_k < 0 || top_k > NX_MAX_TOP_K)
        return set_err(c, NX_INVALID_ARGUMENT, "bad frame shape");
    cudaSetDevice(c->device);
    nx_frame* f = new (std::nothrow) nx_frame;
    if (!f) return set_err(c, NX_OUT_OF_MEMORY, "host allocation");
    f->ctx = c;
    f->device = c->device;
    if (cudaMalloc(&f->stats, sizeof(FrameStatsD)) != cudaSuccess) {
        delete f;
        return set_err(c, NX_OUT_OF_MEMORY, "frame stats");
    }
    cudaMemset(f->stats, 0, sizeof(FrameStatsD));
    if (cudaEventCreateWithFlags(&f->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->ev_busy, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->ev_counts, cudaEventDisableTiming) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&f->h_counts), 2 * sizeof(int32_t), cudaHostAllocDefault) !=
            cudaSuccess) {
        nx_frame_destroy(f);
        return set_err(c, NX_CUDA_ERROR, "frame events");
    }
    int st = frame_shape(c, f, width, height, top_k, 16);
    if (st) {
        nx_frame_destroy(f);
        return st;
    }
    *out = f;
    return NX_OK;
}

void nx_frame_destroy(nx_frame* f) {
    if (!f) return;
    cudaSetDevice(f->device);
    if (f->ev_busy) cudaEventSynchronize(f->ev_busy);  // texture pass / download still reading it
    for (DevBuf* b : {&f->base, &f->ids, &f->depths, &f->weights, &f->texture, &f->final_img, &f->residual,
                      &f->tile_offsets, &f->base64, &f->residual64, &f->tex_f, &f->texture64, &f->final64})
        b->release();
    if (f->stats) cudaFree(f->stats);
    if (f->ev_ready) cudaEventDestroy(f->ev_ready);
    if (f->ev_busy) cudaEventDestroy(f->ev_busy);
    if (f->ev_counts) {
        cudaEventSynchronize(f->ev_counts);
        cudaEventDestroy(f->ev_counts);
    }
    if (f->h_counts) cudaFreeHost(f->h_counts);
    delete f;
}

int nx_frame_view_get(const nx_frame* f, nx_frame_view* v) {
    if (!f || !v) return NX_INVALID_ARGUMENT;
    if (const int st = frame_settle(f->ctx, const_cast<nx_frame*>(f))) return st;
    v->width = f->W;
    v->height = f->H;
    v->top_k = f->K;
    v->tiles_x = f->tiles_x;
    v->tiles_y = f->tiles_y;
    v->base = f->base.as<float>();
    v->ids = f->ids.as<int32_t>();
    v->depths = f->depths.as<double>();
    v->weights = f->weights.as<double>();
    v->texture = f->texture.as<float>();
    v->final_img = f->final_img.as<float>();
    v->residual = f->residual.as<float>();
    return NX_OK;
}

int nx_frame_download(nx_ctx* c, const nx_frame* fc, const nx_host_frame* dst, void* stream) {
    if (!c || !fc || !dst) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    nx_frame* f = const_cast<nx_frame*>(fc);  // only the frame's ordering events change
    if (const int st = frame_settle(c, f)) return st;
    // default: the third (copy) stream, after the frame's texture pass, so that the
    // copy overlaps the next frames' passes on the other two streams
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->stream3;
    NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_ready, 0));
    if (f->busy_pending) NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_busy, 0));
    const size_t npix = static_cast<size_t>(f->W) * f->H, ns = npix * f->K;
    // Pinned, device-mapped destinations take the streaming copy kernel (nx_copy.cu);
    // anything else a DMA memcpy. NX_DOWNLOAD=memcpy forces the DMA engine.
    static const bool force_dma = [] {
        const char* e = std::getenv("NX_DOWNLOAD");
        return e && std::strcmp(e, "memcpy") == 0;
    }();
    CopyJobs jobs{};
    auto cp = [&](void* d, const DevBuf& b, size_t bytes, int narrow = 0) -> cudaError_t {
        if (!d || !bytes) return cudaSuccess;
        if (!force_dma || narrow) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, d) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer &&
                jobs.n < 8) {
                jobs.j[jobs.n++] = {static_cast<const uint8_t*>(b.p), static_cast<uint8_t*>(at.devicePointer), bytes,
                                    narrow};
                return cudaSuccess;
            }
            cudaGetLastError();  // unregistered host memory reports an error here: not fatal
        }
        if (narrow) return cudaErrorInvalidValue;  // the narrowing copy needs pinned (mapped) memory
        return cudaMemcpyAsync(d, b.p, bytes, cudaMemcpyDeviceToHost, s);
    };
    if (dst->weights_f32 && dst->weights)
        return set_err(c, NX_INVALID_ARGUMENT, "weights and weights_f32 are exclusive");
    NX_CUDA(c, cp(dst->base, f->base, npix * 3 * sizeof(float)));
    NX_CUDA(c, cp(dst->ids, f->ids, ns * sizeof(int32_t)));
    NX_CUDA(c, cp(dst->depths, f->depths, ns * sizeof(double)));
    NX_CUDA(c, cp(dst->weights, f->weights, ns * sizeof(double)));
    if (dst->weights_f32 && ns) {
        const int st = cp(dst->weights_f32, f->weights, ns * sizeof(double), 1);
        if (st == cudaErrorInvalidValue)
            return set_err(c, NX_INVALID_ARGUMENT, "weights_f32 needs pinned (cudaHostAlloc / registered) memory");
        NX_CUDA(c, static_cast<cudaError_t>(st));
    }
    NX_CUDA(c, cp(dst->texture, f->texture, ns * 3 * sizeof(float)));
    NX_CUDA(c, cp(dst->final_img, f->final_img, npix * 3 * sizeof(float)));
    NX_CUDA(c, cp(dst->residual, f->residual, npix * sizeof(float)));
    if (dst->base_f64 && f->base64_valid) NX_CUDA(c, cp(dst->base_f64, f->base64, npix * 3 * sizeof(double)));
    if (dst->residual_f64 && f->base64_valid) NX_CUDA(c, cp(dst->residual_f64, f->residual64, npix * sizeof(double)));
    if (dst->texture_f64 && f->f64) NX_CUDA(c, cp(dst->texture_f64, f->texture64, ns * 3 * sizeof(double)));
    if (dst->final_f64 && f->f64) NX_CUDA(c, cp(dst->final_f64, f->final64, npix * 3 * sizeof(double)));
    launch_stream_copy(jobs, s);
    NX_CUDA(c, cudaGetLastError());
    NX_CUDA(c, cudaEventRecord(f->ev_busy, s));
    f->busy_pending = true;
    return NX_OK;
}

int nx_frame_upload(nx_ctx* c, nx_frame* f, int width, int height, int top_k, const nx_host_frame* src,
                    void* stream) {
    if (!c || !f || !src || width < 0 || height < 0 || top_k < 0 || top_k > NX_MAX_TOP_K)
        return set_err(c, NX_INVALID_ARGUMENT, "bad frame upload");
    cudaSetDevice(c->device);
    if (src->base_f64 || src->residual_f64) f->keep_backward = true;
    int st = frame_shape(c, f, width, height, top_k, 16);  // tiles are re-derived by collection_pass
    if (st) return st;
    cudaStream_t s = pick_stream(c, stream);
    const size_t npix = static_cast<size_t>(width) * height, ns = npix * top_k;
    auto cp = [&](DevBuf& b, const void* h, size_t bytes) -> cudaError_t {
        if (!h || !bytes) return cudaSuccess;
        return cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, s);
    };
    NX_CUDA(c, cp(f->base, src->base, npix * 3 * sizeof(float)));
    NX_CUDA(c, cp(f->ids, src->ids, ns * sizeof(int32_t)));
    NX_CUDA(c, cp(f->depths, src->depths, ns * sizeof(double)));
    NX_CUDA(c, cp(f->weights, src->weights, ns * sizeof(double)));
    NX_CUDA(c, cp(f->texture, src->texture, ns * 3 * sizeof(float)));
    NX_CUDA(c, cp(f->final_img, src->final_img, npix * 3 * sizeof(float)));
    NX_CUDA(c, cp(f->residual, src->residual, npix * sizeof(float)));
    if (src->base_f64) {
        NX_CUDA(c, cp(f->base64, src->base_f64, npix * 3 * sizeof(double)));
        f->base64_valid = true;
    }
    NX_CUDA(c, cp(f->residual64, src->residual_f64, npix * sizeof(double)));
    return NX_OK;
}

int nx_frame_stats_get(nx_ctx* c, const nx_frame* f, nx_frame_stats* out) {
    if (!c || !f || !out) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (const int st = frame_settle(c, const_cast<nx_frame*>(f))) return st;
    FrameStatsD h;
    NX_CUDA(c, cudaStreamSynchronize(c->stream));
    NX_CUDA(c, cudaDeviceSynchronize());
    NX_CUDA(c, cudaMemcpy(&h, f->stats, sizeof h, cudaMemcpyDeviceToHost));
    std::memset(out, 0, sizeof *out);
    out->n_nexels = f->n_nexels;
    out->n_dropped_support = static_cast<int64_t>(h.cls[CLS_SUPPORT]);
    out->n_behind = static_cast<int64_t>(h.cls[CLS_BEHIND]);
    out->n_offscreen = static_cast<int64_t>(h.cls[CLS_OFFSCREEN]);
    out->n_rect = static_cast<int64_t>(h.cls[CLS_RECT]);
    out->n_straddlers = static_cast<int64_t>(h.cls[CLS_STRADDLER]);
    out->n_entries = out->n_rect + out->n_straddlers;
    out->n_straddlers_kept = static_cast<int64_t>(h.straddlers_kept);
    out->tile_keys = static_cast<int64_t>(h.tile_keys);
    out->work_keys = static_cast<int64_t>(h.work_keys);
    out->n_queries = static_cast<int64_t>(h.queries);
    out->near_alpha = static_cast<int64_t>(h.near[NEAR_ALPHA]);
    out->near_transmittance = static_cast<int64_t>(h.near[NEAR_TRANSMITTANCE]);
    out->near_topk = static_cast<int64_t>(h.near[NEAR_TOPK]);
    out->near_depth = static_cast<int64_t>(h.near[NEAR_DEPTH]);
    out->near_rect = static_cast<int64_t>(h.near[NEAR_RECT]);
    out->near_support = static_cast<int64_t>(h.near[NEAR_SUPPORT]);
    out->redo_tiles = static_cast<int64_t>(h.redo_tiles);
    return NX_OK;
}

int nx_collection_pass(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, void* stream) {
    if (!c || !f) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    return collection(c, scene, cam, f, pick_stream(c, stream), nullptr, nullptr, 0, 0, 0);
}

int nx_texturing_pass(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, void* stream) {
    if (!c || !f || !scene || !cam) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    return texturing(c, scene, cam, f, stream ? static_cast<cudaStream_t>(stream) : c->stream2);
}

// With the context's own streams the texture pass runs on the second stream, so it
// overlaps the next frame's binning and compositing (into another frame) on the
// first; a frame's reuse and its downloads are ordered by its events.
int nx_render(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, void* stream) {
    if (!c || !f) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = pick_stream(c, stream);
    int st = collection(c, scene, cam, f, s, nullptr, nullptr, 0, 0, 0);
    if (st) return st;
    return texturing(c, scene, cam, f, stream ? s : c->stream2);
}

// A batch of views: cams[i] into frames[i % n_frames], pipelined like back-to-back
// nx_render calls (each frame's texture pass overlaps the next view's collection).
int nx_render_views(nx_ctx* c, const nx_scene* scene, const nx_camera* cams, int n_views, nx_frame* const* frames,
                    int n_frames, void* stream) {
    if (!c || !scene || (n_views > 0 && (!cams || !frames || n_frames < 1)))
        return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    for (int i = 0; i < n_frames && i < n_views; ++i)
        if (!frames[i]) return set_err(c, NX_INVALID_ARGUMENT, "null frame");
    for (int i = 0; i < n_views; ++i)
        if (const int st = nx_render(c, scene, &cams[i], frames[i % n_frames], stream)) return st;
    return NX_OK;
}

int nx_frame_set_backward(nx_ctx* c, nx_frame* f, int enable) {
    if (!c || !f) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    f->keep_backward = enable != 0;
    if (!f->keep_backward) {
        f->base64.release();
        f->base64_valid = false;
        return NX_OK;
    }
    NX_CUDA(c, f->base64.ensure(std::max<size_t>(static_cast<size_t>(f->W) * f->H * 3, 1) * sizeof(double)));
    return NX_OK;
}

// render_backward (renderer.cpp:251-401): field branch, then the reverse march of
// the compositing branch, then activation_backward per primitive.
int nx_render_backward(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f, const nx_upstream* up,
                       const nx_grads* g, const double* err_pixel, double* blended_error, void* stream) {
    if (!c || !f || !up || !g) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    int st;
    if ((st = frame_settle(c, f))) return st;
    if ((st = check_inputs(c, scene, cam, pick_stream(c, stream)))) return st;
    if (!g->prims || !g->table || !g->w1 || !g->w2 || !g->w3)
        return set_err(c, NX_INVALID_ARGUMENT, "render_backward: every gradient array is required");
    if (f->W != cam->width || f->H != cam->height || f->K != scene->st.top_k)
        return set_err(c, NX_INVALID_ARGUMENT, "render_backward: the frame is not the forward output for this camera");
    if (!f->base64_valid)
        return set_err(c, NX_INVALID_ARGUMENT,
                       "render_backward: the frame did not keep the backward state (nx_frame_set_backward before "
                       "collection_pass)");
    cudaSetDevice(c->device);
    cudaStream_t s = pick_stream(c, stream);
    NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_ready, 0));
    if (f->busy_pending) NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_busy, 0));
    if (!c->bwd_lists) {
        if ((st = nx_frame_create(c, 0, 0, 0, &c->bwd_lists))) return st;
    }
    nx_frame* lf = c->bwd_lists;
    lf->tiles_x = (cam->width + scene->st.tile - 1) / scene->st.tile;  // reference tiles (stats only)
    lf->tiles_y = (cam->height + scene->st.tile - 1) / scene->st.tile;
    int64_t total = 0;
    const bool prof = c->profiling;
    c->profiling = false;  // the stage events describe forward frames only
    // 8x8 work tiles (measured at config 2: 6.1 ms vs 6.6 ms with 16x16 — shorter lists per
    // warp; and small images keep enough CTAs); NX_BWD_TILE=16 selects the 16x16 variant
    static const int forced_tile = [] {
        const char* e = std::getenv("NX_BWD_TILE");
        return e ? std::atoi(e) : 0;
    }();
    const int bwd_tile = forced_tile == 16 ? 16 : 8;
    // The reference re-bins here (renderer.cpp:257); the forward's work lists of this frame
    // are the same lists when nothing has rebuilt the shared list buffers since, for the same
    // scene version and camera — then they (and the primitive records) are reused.
    const nx_camera& lc = c->lists_cam;
    const bool same_cam = lc.width == cam->width && lc.height == cam->height && lc.fx == cam->fx &&
                          lc.fy == cam->fy && lc.cx == cam->cx && lc.cy == cam->cy &&
                          std::memcmp(lc.R, cam->R, sizeof lc.R) == 0 && std::memcmp(lc.t, cam->t, sizeof lc.t) == 0;
    const bool reuse = bwd_tile == kWorkTile && f->lists_gen != 0 && f->lists_gen == c->lists_gen &&
                       c->lists_scene == scene && c->lists_scene_version == scene->version &&
                       c->lists_tile == kWorkTile && same_cam;
    if (reuse) {
        lf = f;
    } else {
        st = build_lists(c, scene, *cam, lf, 0, s, &total, bwd_tile);
    }
    c->profiling = prof;
    if (st) return st;

    const int64_t n = scene->n, npix = static_cast<int64_t>(f->W) * f->H, ns = npix * f->K;
    NX_CUDA(c, c->d_t_slot.ensure(std::max<int64_t>(ns, 1) * sizeof(double)));
    NX_CUDA(c, c->act_grad.ensure(std::max<int64_t>(n, 1) * kActFields * sizeof(double)));
    const Xacc pacc{nullptr, std::max<int64_t>(n, 1) * kPrimAccVals};
    NX_CUDA(c, c->xacc_prims.ensure_zeroed(xacc_bytes(pacc.m), s));
    const Xacc prim_acc{c->xacc_prims.as<unsigned long long>(), pacc.m};
    FrameDev fd = frame_dev(f);
    fd.tiles_x = lf->ltiles_x;
    fd.tiles_y = lf->ltiles_y;
    const CamD cd = make_cam(*cam);
    bool join_side = false;  // the field backward forked work onto stream_bwd
    if (f->K > 0) {
        if (up->d_final || up->d_texture) {
            FieldBwdArgs fa;
            fa.scene = scene_dev(scene);
            fa.st = scene->st;
            fa.cam = cd;
            fa.fb = fd;
            fa.d_final = up->d_final;
            fa.d_texture = up->d_texture;
            fa.d_t_slot = c->d_t_slot.as<double>();
            fa.g_table = g->table;
            fa.g_w1 = g->w1;
            fa.g_w2 = g->w2;
            fa.g_w3 = g->w3;
            fa.scratch = &c->field_bwd;
            // NX_BWD_OVERLAP=0: everything on s
            static const bool overlap = [] {
                const char* e = std::getenv("NX_BWD_OVERLAP");
                return !(e && e[0] == '0');
            }();
            if (overlap) {
                fa.side = c->stream_bwd;
                fa.ev_fork = c->ev_bwd_fork;
                fa.ev_join = c->ev_bwd_join;
            }
            if ((st = launch_field_backward(fa, s)))
                return set_err(c, st, "texture field shape not supported by render_backward");
            join_side = overlap;
        } else {
            NX_CUDA(c, cudaMemsetAsync(c->d_t_slot.p, 0, ns * sizeof(double), s));
        }
    }
    CompositeBwdArgs ca;
    ca.rec = c->rec.as<double>();
    ca.recf = c->recf.as<float4>();
    ca.n = std::max<int64_t>(n, 1);
    ca.sh = scene->sh.as<float>();
    ca.list_ids = lf->list_ids.as<int32_t>();
    ca.tile_offsets = lf->tile_offsets.as<int32_t>();
    ca.st = scene->st;
    ca.cam = cd;
    ca.fb = fd;
    ca.sh_degree = scene->st.no_prim_sh ? 0 : 3;
    ca.d_final = up->d_final;
    ca.d_weights = f->K > 0 ? up->d_weights : nullptr;
    ca.d_t_slot = c->d_t_slot.as<double>();
    ca.err_pixel = blended_error ? err_pixel : nullptr;
    ca.acc = prim_acc;
    ca.tile = bwd_tile;
    launch_composite_backward(ca, s);
    launch_prim_finalize(scene_dev(scene), scene->st.no_gamma, prim_acc, c->act_grad.as<double>(), g->prims,
                         err_pixel ? blended_error : nullptr, s);
    if (join_side) NX_CUDA(c, cudaStreamWaitEvent(s, c->ev_bwd_join, 0));
    NX_CUDA(c, cudaEventRecord(f->ev_busy, s));
    f->busy_pending = true;
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

int nx_render_backward_host(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, nx_frame* f,
                            const nx_upstream* up, const nx_grads* g, const double* err_pixel,
                            double* blended_error) {
    if (!c || !f || !up || !g || !scene || !cam) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    int st;
    if ((st = check_inputs(c, scene, cam))) return st;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const size_t npix = static_cast<size_t>(cam->width) * cam->height, K = scene->st.top_k;
    const size_t n = static_cast<size_t>(scene->n);
    const nx_field_desc& fd = scene->field;
    const size_t nin = static_cast<size_t>(fd.levels) * fd.features, nh = fd.n_hidden;
    const size_t g_sizes[5] = {n * NX_PARAMS_PER_NEXEL,
                               static_cast<size_t>(fd.levels) * (size_t(1) << fd.log2_table) * fd.features,
                               nh * nin, nh * nh, NX_SH_VALUES * nh};
    double* g_host[5] = {g->prims, g->table, g->w1, g->w2, g->w3};
    for (double* p : g_host)
        if (!p) return set_err(c, NX_INVALID_ARGUMENT, "render_backward: every gradient array is required");
    nx_grads gd;
    double** g_dev[5] = {&gd.prims, &gd.table, &gd.w1, &gd.w2, &gd.w3};
    for (int i = 0; i < 5; ++i) {
        NX_CUDA(c, c->h_grads[i].ensure(std::max<size_t>(g_sizes[i], 1) * sizeof(double)));
        *g_dev[i] = c->h_grads[i].as<double>();
        NX_CUDA(c, cudaMemcpyAsync(*g_dev[i], g_host[i], g_sizes[i] * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    const double* u_host[3] = {up->d_final, up->d_weights, up->d_texture};
    const size_t u_sizes[3] = {npix * 3, npix * K, npix * K * 3};
    const double* u_dev[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < 3; ++i) {
        if (!u_host[i] || !u_sizes[i]) continue;
        NX_CUDA(c, c->h_up[i].ensure(u_sizes[i] * sizeof(double)));
        NX_CUDA(c, cudaMemcpyAsync(c->h_up[i].p, u_host[i], u_sizes[i] * sizeof(double), cudaMemcpyHostToDevice, s));
        u_dev[i] = c->h_up[i].as<double>();
    }
    nx_upstream ud{u_dev[0], u_dev[1], u_dev[2]};
    double* err_dev = nullptr;
    double* blend_dev = nullptr;
    if (err_pixel && blended_error) {
        NX_CUDA(c, c->h_err.ensure(std::max<size_t>(npix, 1) * sizeof(double)));
        NX_CUDA(c, cudaMemcpyAsync(c->h_err.p, err_pixel, npix * sizeof(double), cudaMemcpyHostToDevice, s));
        NX_CUDA(c, c->h_blend.ensure(std::max<size_t>(n, 1) * sizeof(double)));
        NX_CUDA(c, cudaMemcpyAsync(c->h_blend.p, blended_error, n * sizeof(double), cudaMemcpyHostToDevice, s));
        err_dev = c->h_err.as<double>();
        blend_dev = c->h_blend.as<double>();
    }
    if ((st = nx_render_backward(c, scene, cam, f, &ud, &gd, err_dev, blend_dev, s))) return st;
    for (int i = 0; i < 5; ++i)
        NX_CUDA(c, cudaMemcpyAsync(g_host[i], *g_dev[i], g_sizes[i] * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (blend_dev)
        NX_CUDA(c, cudaMemcpyAsync(blended_error, blend_dev, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    return NX_OK;
}

void nx_loss_weights_default(nx_loss_weights* w) {  // LossWeights (losses.hpp:12-18)
    if (!w) return;
    w->dssim = 0.2;
    w->alpha = 0.005;
    w->texture = 0.5;
    w->opacity = 0.01;
    w->grid = 0.01;
}

// losses_backward (losses.cpp:107-238) on the frame's final_img / slots.
}  // extern "C"
namespace {
int losses_backward(nx_ctx* c, const nx_scene* scene, const nx_frame* fc, const double* gt,
                    const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                    const nx_grads* g, nx_loss_terms* terms, void* stream, const double* table64) {
    if (!c || !scene || !fc || !gt || !w || !d_final || !g || !g->prims || !g->table || !terms)
        return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    nx_frame* f = const_cast<nx_frame*>(fc);
    if (const int st = frame_settle(c, f)) return st;
    if (f->K > 0 && (!d_weights || !d_texture))
        return set_err(c, NX_INVALID_ARGUMENT, "losses_backward: d_weights / d_texture are required when top_k > 0");
    if (f->K != scene->st.top_k)
        return set_err(c, NX_INVALID_ARGUMENT, "losses_backward: the frame does not match the scene's top_k");
    cudaSetDevice(c->device);
    cudaStream_t s = pick_stream(c, stream);
    NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_ready, 0));
    if (f->busy_pending) NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_busy, 0));
    const int64_t npix = static_cast<int64_t>(f->W) * f->H;
    NX_CUDA(c, c->loss_scratch.ensure(losses_scratch_bytes(npix)));
    const int st = launch_losses_backward(scene_dev(scene), frame_dev(f), gt, *w, d_final, d_weights, d_texture,
                                          g->prims, g->table, terms, c->loss_scratch.p, s, table64);
    if (st) return set_err(c, st, "losses_backward: field shape not supported");
    NX_CUDA(c, cudaEventRecord(f->ev_busy, s));
    f->busy_pending = true;
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}
}  // namespace
extern "C" {

int nx_losses_backward(nx_ctx* c, const nx_scene* scene, const nx_frame* fc, const double* gt,
                       const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                       const nx_grads* g, nx_loss_terms* terms, void* stream) {
    return losses_backward(c, scene, fc, gt, w, d_final, d_weights, d_texture, g, terms, stream, nullptr);
}

int nx_pixel_error(nx_ctx* c, const nx_frame* fc, const double* gt, double* err, void* stream) {
    if (!c || !fc || !gt || !err) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    nx_frame* f = const_cast<nx_frame*>(fc);
    if (const int st = frame_settle(c, f)) return st;
    cudaSetDevice(c->device);
    cudaStream_t s = pick_stream(c, stream);
    NX_CUDA(c, cudaStreamWaitEvent(s, f->ev_ready, 0));
    launch_pixel_error(frame_dev(f).final_img, gt, static_cast<int64_t>(f->W) * f->H, err, s);
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

int nx_losses_backward_host(nx_ctx* c, const nx_scene* scene, const nx_frame* fc, const double* gt,
                            const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                            const nx_grads* g, nx_loss_terms* terms) {
    if (!c || !scene || !fc || !gt || !w || !d_final || !g || !g->prims || !g->table || !terms)
        return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const size_t npix = static_cast<size_t>(fc->W) * fc->H, K = fc->K, n = static_cast<size_t>(scene->n);
    const nx_field_desc& fd = scene->field;
    const size_t ntab = static_cast<size_t>(fd.levels) * (size_t(1) << fd.log2_table) * fd.features;
    // device copies: gt, outputs (d_final, d_weights, d_texture), grads (prims, table), terms
    NX_CUDA(c, c->h_gt.ensure(std::max<size_t>(npix * 3, 1) * sizeof(double)));
    NX_CUDA(c, cudaMemcpyAsync(c->h_gt.p, gt, npix * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
    const size_t u_sizes[3] = {npix * 3, npix * K, npix * K * 3};
    double* u_host[3] = {d_final, d_weights, d_texture};
    for (int i = 0; i < 3; ++i) NX_CUDA(c, c->h_up[i].ensure(std::max<size_t>(u_sizes[i], 1) * sizeof(double)));
    const size_t g_sizes[2] = {n * NX_PARAMS_PER_NEXEL, ntab};
    double* g_host[2] = {g->prims, g->table};
    for (int i = 0; i < 2; ++i) {
        NX_CUDA(c, c->h_grads[i].ensure(std::max<size_t>(g_sizes[i], 1) * sizeof(double)));
        NX_CUDA(c, cudaMemcpyAsync(c->h_grads[i].p, g_host[i], g_sizes[i] * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    NX_CUDA(c, c->h_terms.ensure(sizeof(nx_loss_terms)));
    nx_grads gd{c->h_grads[0].as<double>(), c->h_grads[1].as<double>(), nullptr, nullptr, nullptr};
    int st = nx_losses_backward(c, scene, fc, c->h_gt.as<double>(), w, c->h_up[0].as<double>(),
                                K ? c->h_up[1].as<double>() : nullptr, K ? c->h_up[2].as<double>() : nullptr, &gd,
                                c->h_terms.as<nx_loss_terms>(), s);
    if (st) return st;
    for (int i = 0; i < 3; ++i)
        if (u_host[i] && u_sizes[i])
            NX_CUDA(c, cudaMemcpyAsync(u_host[i], c->h_up[i].p, u_sizes[i] * sizeof(double), cudaMemcpyDeviceToHost, s));
    for (int i = 0; i < 2; ++i)
        NX_CUDA(c, cudaMemcpyAsync(g_host[i], c->h_grads[i].p, g_sizes[i] * sizeof(double), cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaMemcpyAsync(terms, c->h_terms.p, sizeof(nx_loss_terms), cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    return NX_OK;
}

// ---------------------------------------------------------------- Adam (adam.cpp, trainer.cpp:238-323)
}  // extern "C"

struct nx_optimizer {
    nx_ctx* ctx = nullptr;
    int device = 0;  // the creating context's device
    int64_t n = 0;
    DevBuf m[NX_NUM_GROUPS], v[NX_NUM_GROUPS];
    DevBuf master[NX_NUM_GROUPS];  // fp64 values of the groups the scene stores in fp32 (5..10)
    DevBuf m_spare[7], v_spare[7], master_spare[7];  // per-nexel rows rebuilt by density control
    int64_t step[NX_NUM_GROUPS] = {};
    int64_t size[NX_NUM_GROUPS] = {};
};

extern "C" {

int nx_optimizer_create(nx_ctx* c, const nx_scene* scene, nx_optimizer** out) {
    if (!c || !scene || !out) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (scene->sh64.p) return set_err(c, NX_UNSUPPORTED, "NX_PRECISION_F64 scenes are render-only (no optimizer)");
    cudaSetDevice(c->device);
    nx_optimizer* o = new (std::nothrow) nx_optimizer;
    if (!o) return set_err(c, NX_OUT_OF_MEMORY, "host allocation");
    o->ctx = c;
    o->device = c->device;
    o->n = scene->n;
    adam_group_sizes(scene_dev(scene), o->size);
    for (int gi = 0; gi < NX_NUM_GROUPS; ++gi) {
        const size_t bytes = std::max<int64_t>(o->size[gi], 1) * sizeof(double);
        if (o->m[gi].ensure(bytes) != cudaSuccess || o->v[gi].ensure(bytes) != cudaSuccess ||
            cudaMemset(o->m[gi].p, 0, bytes) != cudaSuccess || cudaMemset(o->v[gi].p, 0, bytes) != cudaSuccess ||
            (gi >= NX_GROUP_SH_DC && o->master[gi].ensure(bytes) != cudaSuccess)) {
            nx_optimizer_destroy(o);
            return set_err(c, NX_OUT_OF_MEMORY, "optimizer state");
        }
    }
    nx_scene* sc = const_cast<nx_scene*>(scene);
    for (int gi = NX_GROUP_SH_DC; gi < NX_NUM_GROUPS; ++gi)
        launch_group_io(gi, scene_dev(scene), sc->geom.as<double>(), sc->sh.as<float>(), sc->table.as<float>(),
                        sc->w1.as<float>(), sc->w2.as<float>(), sc->w3.as<float>(), o->master[gi].as<double>(), true,
                        c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
        nx_optimizer_destroy(o);
        return set_err(c, NX_CUDA_ERROR, "optimizer masters");
    }
    *out = o;
    return NX_OK;
}

int nx_losses_backward_opt(nx_ctx* c, const nx_scene* scene, const nx_frame* fc, const double* gt,
                           const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                           const nx_grads* g, nx_loss_terms* terms, const nx_optimizer* opt, void* stream) {
    const double* table64 = nullptr;
    if (opt) {
        const nx_field_desc& fd = scene ? scene->field : nx_field_desc{};
        const int64_t ntab = static_cast<int64_t>(fd.levels) * (int64_t(1) << fd.log2_table) * fd.features;
        if (opt->size[NX_GROUP_GRID] != ntab)
            return set_err(c, NX_INVALID_ARGUMENT, "losses_backward: the optimizer does not match the scene's table");
        table64 = opt->master[NX_GROUP_GRID].as<double>();
    }
    return losses_backward(c, scene, fc, gt, w, d_final, d_weights, d_texture, g, terms, stream, table64);
}

int nx_optimizer_size(const nx_optimizer* o, int group, int64_t* count) {
    if (!o || !count || group < 0 || group >= NX_NUM_GROUPS) return NX_INVALID_ARGUMENT;
    *count = o->size[group];
    return NX_OK;
}

int nx_optimizer_set_params(nx_ctx* c, nx_optimizer* o, nx_scene* scene, int group, const double* host,
                            int64_t count) {
    if (!c || !o || !scene || !host) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (group < 0 || group >= NX_NUM_GROUPS || count != o->size[group] || scene->n != o->n)
        return set_err(c, NX_INVALID_ARGUMENT, "optimizer_set_params: bad group or size");
    if (count == 0) return NX_OK;
    cudaSetDevice(c->device);
    scene->version = next_scene_version();
    cudaStream_t s = c->stream;
    DevBuf rows;
    NX_CUDA(c, rows.ensure(count * sizeof(double)));
    NX_CUDA(c, cudaMemcpyAsync(rows.p, host, count * sizeof(double), cudaMemcpyHostToDevice, s));
    // the scene's copy (geometry: the values themselves; fp32 groups: their rounding)
    launch_group_io(group, scene_dev(scene), scene->geom.as<double>(), scene->sh.as<float>(), scene->table.as<float>(),
                    scene->w1.as<float>(), scene->w2.as<float>(), scene->w3.as<float>(), rows.as<double>(), false, s);
    if (group >= NX_GROUP_SH_DC)
        NX_CUDA(c, cudaMemcpyAsync(o->master[group].p, rows.p, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    return NX_OK;
}

int nx_optimizer_download(nx_ctx* c, const nx_optimizer* o, const nx_scene* scene, int group, double* params,
                          double* m, double* v) {
    if (!c || !o || !scene) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (group < 0 || group >= NX_NUM_GROUPS || scene->n != o->n)
        return set_err(c, NX_INVALID_ARGUMENT, "optimizer_download: bad group or scene");
    const int64_t count = o->size[group];
    if (count == 0) return NX_OK;
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    NX_CUDA(c, cudaStreamSynchronize(s));
    if (params) {
        if (group >= NX_GROUP_SH_DC) {
            NX_CUDA(c, cudaMemcpy(params, o->master[group].p, count * sizeof(double), cudaMemcpyDeviceToHost));
        } else {
            DevBuf rows;
            NX_CUDA(c, rows.ensure(count * sizeof(double)));
            nx_scene* sc = const_cast<nx_scene*>(scene);
            launch_group_io(group, scene_dev(scene), sc->geom.as<double>(), sc->sh.as<float>(), sc->table.as<float>(),
                            sc->w1.as<float>(), sc->w2.as<float>(), sc->w3.as<float>(), rows.as<double>(), true, s);
            NX_CUDA(c, cudaMemcpyAsync(params, rows.p, count * sizeof(double), cudaMemcpyDeviceToHost, s));
            NX_CUDA(c, cudaStreamSynchronize(s));
        }
    }
    if (m) NX_CUDA(c, cudaMemcpy(m, o->m[group].p, count * sizeof(double), cudaMemcpyDeviceToHost));
    if (v) NX_CUDA(c, cudaMemcpy(v, o->v[group].p, count * sizeof(double), cudaMemcpyDeviceToHost));
    return NX_OK;
}

void nx_optimizer_destroy(nx_optimizer* o) {
    if (!o) return;
    cudaSetDevice(o->device);
    for (int gi = 0; gi < NX_NUM_GROUPS; ++gi) {
        o->m[gi].release();
        o->v[gi].release();
        o->master[gi].release();
    }
    for (int gi = 0; gi < 7; ++gi) {
        o->m_spare[gi].release();
        o->v_spare[gi].release();
        o->master_spare[gi].release();
    }
    delete o;
}

int nx_optimizer_steps(const nx_optimizer* o, int64_t* steps) {
    if (!o || !steps) return NX_INVALID_ARGUMENT;
    for (int gi = 0; gi < NX_NUM_GROUPS; ++gi) steps[gi] = o->step[gi];
    return NX_OK;
}

int nx_optimizer_step(nx_ctx* c, nx_optimizer* o, nx_scene* scene, const nx_grads* g, const nx_adam_config* cfg,
                      void* stream) {
    if (!c || !o || !scene || !g || !cfg || !g->prims || !g->table || !g->w1 || !g->w2 || !g->w3)
        return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (scene->n != o->n) return set_err(c, NX_INVALID_ARGUMENT, "optimizer_step: the scene changed size");
    cudaSetDevice(c->device);
    cudaStream_t s = pick_stream(c, stream);
    scene->version = next_scene_version();
    const SceneDev sd = scene_dev(scene);
    for (int gi = 0; gi < NX_NUM_GROUPS; ++gi) {
        if (cfg[gi].lr < 0.0) continue;
        ++o->step[gi];  // adam.cpp:12: the step counts even when the group is empty
        if (o->size[gi] == 0) continue;
        launch_adam_group(gi, sd, scene->geom.as<double>(), scene->sh.as<float>(), scene->table.as<float>(),
                          scene->w1.as<float>(), scene->w2.as<float>(), scene->w3.as<float>(), *g, o->m[gi].as<double>(),
                          o->v[gi].as<double>(), gi >= NX_GROUP_SH_DC ? o->master[gi].as<double>() : nullptr, cfg[gi],
                          o->step[gi], s);
    }
    NX_CUDA(c, cudaGetLastError());
    return NX_OK;
}

// ---------------------------------------------------------------- density control
namespace {
constexpr int kRowWidth[7] = {3, 4, 2, 1, 2, 3, 45};  // per-nexel Adam groups (trainer.cpp kRowWidth)

// Rebuilds the scene (and the optimizer's per-nexel rows) in the layout of n_new nexels
// from new_to_old (device), into the spare buffers that are then swapped in (no
// allocation once they have grown): geometry already in scene->geom_spare when
// geom_done (densify), else gathered; SH already in scene->sh (swapped) when sh_done. Moments follow new_to_old (-1: fresh zeros,
// adam_remap_rows); the SH masters follow src_rows (the row each new row's values come
// from: a split child's parent), new_to_old when null.
int apply_row_map(nx_ctx* c, nx_scene* scene, nx_optimizer* opt, int64_t n_new, const int32_t* n2o,
                  bool geom_done, bool sh_done, cudaStream_t s, const int32_t* src_rows = nullptr) {
    const int64_t n = scene->n;
    if (!geom_done) {
        NX_CUDA(c, scene->geom_spare.ensure(std::max<int64_t>(n_new, 1) * kGeomFields * sizeof(double)));
        launch_gather_geom(scene->geom.as<double>(), n, scene->geom_spare.as<double>(), n_new, n2o, s);
    }
    if (!sh_done) {
        NX_CUDA(c, scene->sh_spare.ensure(std::max<int64_t>(n_new, 1) * NX_SH_VALUES * sizeof(float)));
        launch_gather_rows_f32(scene->sh.as<float>(), scene->sh_spare.as<float>(), n_new, NX_SH_VALUES, n2o, s);
    }
    if (opt) {
        for (int gi = 0; gi < 7; ++gi) {
            const size_t bytes = std::max<int64_t>(n_new * kRowWidth[gi], 1) * sizeof(double);
            NX_CUDA(c, opt->m_spare[gi].ensure(bytes));
            NX_CUDA(c, opt->v_spare[gi].ensure(bytes));
            launch_gather_rows_f64(opt->m[gi].as<double>(), opt->m_spare[gi].as<double>(), n_new, kRowWidth[gi], n2o, s);
            launch_gather_rows_f64(opt->v[gi].as<double>(), opt->v_spare[gi].as<double>(), n_new, kRowWidth[gi], n2o, s);
            if (gi >= NX_GROUP_SH_DC) {
                NX_CUDA(c, opt->master_spare[gi].ensure(bytes));
                launch_gather_rows_f64(opt->master[gi].as<double>(), opt->master_spare[gi].as<double>(), n_new,
                                       kRowWidth[gi], src_rows ? src_rows : n2o, s);
            }
        }
    }
    NX_CUDA(c, cudaStreamSynchronize(s));
    if (opt) {
        for (int gi = 0; gi < 7; ++gi) {
            std::swap(opt->m[gi], opt->m_spare[gi]);
            std::swap(opt->v[gi], opt->v_spare[gi]);
            if (gi >= NX_GROUP_SH_DC) std::swap(opt->master[gi], opt->master_spare[gi]);
            opt->size[gi] = n_new * kRowWidth[gi];
        }
        opt->n = n_new;
    }
    std::swap(scene->geom, scene->geom_spare);
    if (!sh_done) std::swap(scene->sh, scene->sh_spare);
    scene->n = n_new;
    scene->version = next_scene_version();
    return NX_OK;
}
}  // namespace

int nx_scene_prune(nx_ctx* c, nx_scene* scene, nx_optimizer* opt, double min_opacity, int32_t* new_to_old,
                   int64_t* n_out) {
    if (!c || !scene) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (scene->sh64.p) return set_err(c, NX_UNSUPPORTED, "NX_PRECISION_F64 scenes are render-only (no pruning)");
    if (opt && opt->n != scene->n) return set_err(c, NX_INVALID_ARGUMENT, "prune: optimizer and scene disagree");
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const int64_t n = scene->n, nn = std::max<int64_t>(n, 1);
    NX_CUDA(c, c->flag.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->pos.ensure(nn * sizeof(int32_t)));
    NX_CUDA(c, c->scratch.ensure((scan_scratch_ints(nn) + 64) * sizeof(int32_t)));
    int32_t* d_total = c->scratch.as<int32_t>();
    launch_prune_flags(scene->geom.as<double>(), n, min_opacity, c->flag.as<int32_t>(), s);
    scan_exclusive(c->flag.as<int32_t>(), c->pos.as<int32_t>(), n, d_total, d_total + 64, s);
    int32_t kept = 0;
    NX_CUDA(c, cudaMemcpyAsync(&kept, d_total, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    if (n == 0) kept = 0;
    DevBuf& map = c->dens_map;
    NX_CUDA(c, map.ensure(std::max<int64_t>(kept, 1) * sizeof(int32_t)));
    launch_compact_map(c->flag.as<int32_t>(), c->pos.as<int32_t>(), n, map.as<int32_t>(), s);
    int st = apply_row_map(c, scene, opt, kept, map.as<int32_t>(), false, false, s);
    if (st) return st;
    if (new_to_old && kept)
        NX_CUDA(c, cudaMemcpyAsync(new_to_old, map.p, kept * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    if (n_out) *n_out = kept;
    return NX_OK;
}

int nx_scene_densify_split(nx_ctx* c, nx_scene* scene, nx_optimizer* opt, const double* errors,
                           const double* uniforms, int64_t budget, double split_fraction, int32_t* new_to_old,
                           int64_t* n_out, int64_t* split_count) {
    if (!c || !scene || !errors || !uniforms) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    if (scene->sh64.p) return set_err(c, NX_UNSUPPORTED, "NX_PRECISION_F64 scenes are render-only (no densify)");
    if (opt && opt->n != scene->n) return set_err(c, NX_INVALID_ARGUMENT, "densify: optimizer and scene disagree");
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const int64_t n = scene->n;
    if (split_count) *split_count = 0;
    if (n_out) *n_out = n;
    int64_t allowed = std::min<int64_t>(static_cast<int64_t>(std::ceil(split_fraction * static_cast<double>(n))),
                                        budget - n);  // density.cpp:109
    auto identity = [&]() -> int {
        if (new_to_old && n) {
            std::vector<int32_t> id(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) id[i] = static_cast<int32_t>(i);
            NX_CUDA(c, cudaMemcpyAsync(new_to_old, id.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            NX_CUDA(c, cudaStreamSynchronize(s));
        }
        return NX_OK;
    };
    if (n == 0 || allowed <= 0) return identity();
    const int64_t nn = std::max<int64_t>(n, 1);
    NX_CUDA(c, c->skeys_a.ensure(nn * sizeof(uint64_t)));
    NX_CUDA(c, c->skeys_b.ensure(nn * sizeof(uint64_t)));
    NX_CUDA(c, c->sids_a.ensure(nn * sizeof(uint32_t)));
    NX_CUDA(c, c->sids_b.ensure(nn * sizeof(uint32_t)));
    NX_CUDA(c, c->scratch.ensure((radix_scratch_ints64(nn) + 64) * sizeof(int32_t)));
    unsigned long long* d_count = reinterpret_cast<unsigned long long*>(c->scratch.as<int32_t>());
    NX_CUDA(c, cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
    launch_split_keys(errors, uniforms, n, c->skeys_a.as<uint64_t>(), c->sids_a.as<uint32_t>(), d_count, s);
    const bool in_b = radix_sort_pairs_u64(c->skeys_a.as<uint64_t>(), c->sids_a.as<uint32_t>(),
                                           c->skeys_b.as<uint64_t>(), c->sids_b.as<uint32_t>(), n, nullptr, 0, 64,
                                           c->scratch.as<int32_t>() + 64, s);
    unsigned long long n_keys = 0;
    NX_CUDA(c, cudaMemcpyAsync(&n_keys, d_count, sizeof n_keys, cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    allowed = std::min<int64_t>(allowed, static_cast<int64_t>(n_keys));
    if (allowed <= 0) return identity();
    std::vector<int32_t> parents(static_cast<size_t>(allowed));
    NX_CUDA(c, cudaMemcpyAsync(parents.data(), in_b ? c->sids_b.p : c->sids_a.p, allowed * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    std::sort(parents.begin(), parents.end());  // density.cpp:132-134
    const int64_t n_new = n + allowed;
    DevBuf &d_par = c->dens_par, &map = c->dens_map, &src = c->dens_src;
    NX_CUDA(c, d_par.ensure(allowed * sizeof(int32_t)));
    NX_CUDA(c, cudaMemcpyAsync(d_par.p, parents.data(), allowed * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    NX_CUDA(c, map.ensure(n_new * sizeof(int32_t)));
    NX_CUDA(c, scene->geom_spare.ensure(n_new * kGeomFields * sizeof(double)));
    NX_CUDA(c, scene->sh_spare.ensure(n_new * NX_SH_VALUES * sizeof(float)));
    NX_CUDA(c, cudaMemcpyAsync(scene->sh_spare.p, scene->sh.p, n * NX_SH_VALUES * sizeof(float),
                               cudaMemcpyDeviceToDevice, s));
    launch_split_children(scene->geom_spare.as<double>(), n_new, scene->geom.as<double>(), n,
                          scene->sh_spare.as<float>(), d_par.as<int32_t>(), allowed, map.as<int32_t>(), s);
    std::swap(scene->sh, scene->sh_spare);
    if (opt) {  // the SH masters' source rows: kept rows themselves, a child its parent
        std::vector<int32_t> h(static_cast<size_t>(n_new));
        for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int32_t>(i);
        for (int64_t r = 0; r < allowed; ++r) h[n + r] = parents[r];
        NX_CUDA(c, src.ensure(n_new * sizeof(int32_t)));
        NX_CUDA(c, cudaMemcpyAsync(src.p, h.data(), n_new * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    int st = apply_row_map(c, scene, opt, n_new, map.as<int32_t>(), true, true, s, opt ? src.as<int32_t>() : nullptr);
    if (st) return st;
    if (new_to_old)
        NX_CUDA(c, cudaMemcpyAsync(new_to_old, map.p, n_new * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    NX_CUDA(c, cudaStreamSynchronize(s));
    if (n_out) *n_out = n_new;
    if (split_count) *split_count = allowed;
    return NX_OK;
}

int nx_scene_download(nx_ctx* c, const nx_scene* scene, double* nexels, double* table, double* w1, double* w2,
                      double* w3) {
    if (!c || !scene) return set_err(c, NX_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(c->device);
    NX_CUDA(c, cudaDeviceSynchronize());
    const int64_t n = scene->n, nn = std::max<int64_t>(n, 1);
    if (nexels && n > 0) {
        std::vector<double> geom(static_cast<size_t>(kGeomFields * nn));
        std::vector<float> sh(static_cast<size_t>(NX_SH_VALUES * nn));
        NX_CUDA(c, cudaMemcpy(geom.data(), scene->geom.p, geom.size() * sizeof(double), cudaMemcpyDeviceToHost));
        NX_CUDA(c, cudaMemcpy(sh.data(), scene->sh.p, sh.size() * sizeof(float), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i) {
            double* p = nexels + i * NX_PARAMS_PER_NEXEL;
            for (int k = 0; k < kGeomFields; ++k) p[k] = geom[k * nn + i];
            for (int k = 0; k < NX_SH_VALUES; ++k) p[12 + k] = sh[i * NX_SH_VALUES + k];
        }
    }
    const nx_field_desc& fd = scene->field;
    const size_t nin = static_cast<size_t>(fd.levels) * fd.features, nh = fd.n_hidden;
    const size_t sizes[4] = {static_cast<size_t>(fd.levels) * (size_t(1) << fd.log2_table) * fd.features, nh * nin,
                             nh * nh, NX_SH_VALUES * nh};
    double* dst[4] = {table, w1, w2, w3};
    const DevBuf* src[4] = {&scene->table, &scene->w1, &scene->w2, &scene->w3};
    for (int k = 0; k < 4; ++k) {
        if (!dst[k]) continue;
        std::vector<float> tmp(sizes[k]);
        NX_CUDA(c, cudaMemcpy(tmp.data(), src[k]->p, sizes[k] * sizeof(float), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < sizes[k]; ++i) dst[k][i] = tmp[i];
    }
    return NX_OK;
}

int nx_debug_tile_lists(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, int reference_lists,
                        int64_t* offsets, int32_t* ids, int64_t capacity, int64_t* total, int32_t* tiles_x,
                        int32_t* tiles_y) {
    int st;
    if ((st = check_inputs(c, scene, cam))) return st;
    nx_frame* f = nullptr;
    if ((st = nx_frame_create(c, cam->width, cam->height, scene->st.top_k, &f))) return st;
    st = frame_shape(c, f, cam->width, cam->height, scene->st.top_k, scene->st.tile);
    int64_t n_keys = 0;
    cudaStream_t s = c->stream;
    if (!st) st = build_lists(c, scene, *cam, f, reference_lists, s, &n_keys);
    if (!st) {
        const int64_t n_tiles = static_cast<int64_t>(f->ltiles_x) * f->ltiles_y;
        std::vector<int32_t> off(static_cast<size_t>(n_tiles + 1));
        cudaError_t e = cudaMemcpyAsync(off.data(), f->tile_offsets.p, off.size() * sizeof(int32_t),
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && ids && n_keys > 0)
            e = cudaMemcpyAsync(ids, f->list_ids.p, std::min(capacity, n_keys) * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_err(c, e, "debug download");
        if (!st && offsets)
            for (int64_t t = 0; t <= n_tiles; ++t) offsets[t] = off[t];
        if (total) *total = n_keys;
        if (tiles_x) *tiles_x = f->ltiles_x;
        if (tiles_y) *tiles_y = f->ltiles_y;
    }
    nx_frame_destroy(f);
    return st;
}

int nx_debug_pixel_hits(nx_ctx* c, const nx_scene* scene, const nx_camera* cam, int y0, int y1, int max_hits,
                        int32_t* hits, int32_t* counts) {
    int st;
    if ((st = check_inputs(c, scene, cam))) return st;
    if (y0 < 0 || y1 > cam->height || y1 < y0 || max_hits < 1 || !hits || !counts)
        return set_err(c, NX_INVALID_ARGUMENT, "bad debug row range");
    const size_t q = static_cast<size_t>(y1 - y0) * cam->width;
    NX_CUDA(c, c->dbg_hits.ensure(std::max<size_t>(q * max_hits, 1) * sizeof(int32_t)));
    NX_CUDA(c, c->dbg_counts.ensure(std::max<size_t>(q, 1) * sizeof(int32_t)));
    nx_frame* f = nullptr;
    if ((st = nx_frame_create(c, cam->width, cam->height, scene->st.top_k, &f))) return st;
    cudaStream_t s = c->stream;
    NX_CUDA(c, cudaMemsetAsync(c->dbg_hits.p, 0xff, q * max_hits * sizeof(int32_t), s));  // -1 = no hit
    NX_CUDA(c, cudaMemsetAsync(c->dbg_counts.p, 0, q * sizeof(int32_t), s));
    st = collection(c, scene, cam, f, s, c->dbg_hits.as<int32_t>(), c->dbg_counts.as<int32_t>(), y0, y1, max_hits);
    if (!st) {
        cudaError_t e = cudaMemcpyAsync(hits, c->dbg_hits.p, q * max_hits * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(counts, c->dbg_counts.p, q * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_err(c, e, "debug download");
    }
    nx_frame_destroy(f);
    return st;
}

}  // extern "C"
