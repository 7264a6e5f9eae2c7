// Drop-in replacement for nexel::train and nexel::mean_psnr (proj/core/src/trainer.cpp:
// 215-349, include/nexel/trainer.hpp:95-101): the reference's training loop with every
// per-iteration step on the sm_100a library through its C-ABI
// (include/nexel_b200.h) — render, losses_backward, the per-pixel error,
// render_backward, Adam over the 11 parameter groups and density control — while
// the scene, the optimizer state (fp64 moments and fp64 master parameters) and the
// ground-truth images of the train views stay resident on the device for the run.
//
// Kept on the host, and taken from the reference itself (trainer.cpp compiled in
// place with `train` renamed, see the Makefile's dropin target): config parsing,
// initialize_scene (the one-time seed-cloud initialisation) and the random stream.
// std::mt19937_64(cfg.seed) is consumed exactly as the reference consumes it —
// initialize_scene, then one std::shuffle of the train views per epoch and one
// uniform per nexel for every densify_split that samples (density.cpp:117-121) —
// so the view order and the split selections follow the reference's.
//
// Semantics kept: the validation codes and messages of train (trainer.cpp:262-267),
// the hooks (on_iteration with the iteration's wall time, on_eval on schedule and at
// the end), the non-finite-loss snapshot (save_checkpoint) and failure, the
// position learning-rate decay, the densify window, and the TrainResult contents
// (scene, extra.cameras / iteration, one AdamState per group — empty moments for a
// group that never stepped — and last_loss). Every reduction on the device is
// order-independent, so two runs give bit-identical results (test_train.cpp
// "training is deterministic run to run").
//
// Data parallelism over views (dp_b200.hpp, NEXEL_DP_WORLD > 1): rank r trains on
// position r of each iteration's `world` positions of the epoch stream (every rank
// consumes the random stream identically), the gradients and the loss terms are averaged
// across the ranks on the device before the Adam step, and the blended errors are summed
// before density control, so every rank holds the same scene; with one rank the loop is
// the reference's.
#include "nexel/trainer.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "nexel/error.hpp"
#include "nexel/metrics.hpp"
#include "nexel/renderer.hpp"
#include "../../include/nexel_b200.h"
#include "dp_b200.hpp"

namespace nexel {

namespace {

static_assert(sizeof(Nexel) == NX_PARAMS_PER_NEXEL * sizeof(double), "Nexel = 60 doubles");
constexpr int kGroupCols[7][2] = {{0, 3}, {3, 4}, {7, 2}, {9, 1}, {10, 2}, {12, 3}, {15, 45}};  // Nexel columns

// Device allocations of one run (freed on every exit path).
struct DevArena {
    std::vector<void*> ptrs;
    ~DevArena() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess)
            fail("out-of-memory", "train: device allocation of " + std::to_string(count * sizeof(T)) + " bytes");
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    void release(void* p) {
        auto it = std::find(ptrs.begin(), ptrs.end(), p);
        if (it != ptrs.end()) {
            cudaFree(p);
            ptrs.erase(it);
        }
    }
};

struct Run {
    nx_ctx* ctx = nullptr;
    nx_scene* scene = nullptr;
    nx_frame* frame = nullptr;
    nx_optimizer* opt = nullptr;
    ~Run() {
        if (opt) nx_optimizer_destroy(opt);
        if (frame) nx_frame_destroy(frame);
        if (scene) nx_scene_destroy(scene);
        if (ctx) nx_ctx_destroy(ctx);
    }
    void check(int status) const {
        if (status == NX_OK) return;
        int st = status;
        const char* msg = ctx ? nx_ctx_last_error(ctx, &st) : "no CUDA context";
        fail(nx_status_name(status), msg);
    }
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail("cuda-error", std::string(what) + ": " + cudaGetErrorString(e));
}

nx_settings to_nx(const RenderSettings& r) {
    nx_settings s;
    std::memset(&s, 0, sizeof s);
    s.top_k = r.top_k;
    s.tile = r.tile;
    for (int c = 0; c < 3; ++c) s.background[c] = r.background[c];
    s.near_eps = r.near_eps;
    s.alpha_max = r.alpha_max;
    s.min_transmittance = r.min_transmittance;
    s.no_gamma = r.no_gamma;
    s.no_prim_sh = r.no_prim_sh;
    s.no_downweight = r.no_downweight;
    return s;
}

nx_camera to_nx(const Camera& c) {
    nx_camera o;
    std::memset(&o, 0, sizeof o);
    o.width = c.width;
    o.height = c.height;
    o.fx = c.fx;
    o.fy = c.fy;
    o.cx = c.cx;
    o.cy = c.cy;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) o.R[r * 3 + k] = c.R.m[r][k];
        o.t[r] = c.t[r];
    }
    return o;
}

LossTerms from_nx(const nx_loss_terms& t) {
    LossTerms o;
    o.l1 = t.l1;
    o.dssim = t.dssim;
    o.image = t.image;
    o.texture = t.texture;
    o.alpha = t.alpha;
    o.opacity = t.opacity;
    o.grid = t.grid;
    o.total = t.total;
    return o;
}

// A group's parameters of the host scene in the optimizer's row layout.
std::vector<double> group_rows(const Scene& s, int g) {
    if (g < 7) {
        const size_t n = s.nexels.size();
        const int c0 = kGroupCols[g][0], w = kGroupCols[g][1];
        std::vector<double> rows(n * w);
        for (size_t i = 0; i < n; ++i) {
            const double* p = &s.nexels[i].mu.x;
            for (int k = 0; k < w; ++k) rows[i * w + k] = p[c0 + k];
        }
        return rows;
    }
    const std::vector<double>* src[4] = {&s.field.grid.table, &s.field.mlp.w1, &s.field.mlp.w2, &s.field.mlp.w3};
    return *src[g - 7];
}

// The device run's parameters (fp64 masters / geometry) back into a host Scene shaped
// like `like` (field configuration, settings, extent).
Scene download_scene(const Run& r, const Scene& like) {
    Scene s = like;
    int64_t rows = 0;
    r.check(nx_optimizer_size(r.opt, kGroupQuat, &rows));
    const size_t n = static_cast<size_t>(rows / 4);
    s.nexels.assign(n, Nexel{});
    for (int g = 0; g < kGroupCount; ++g) {
        int64_t count = 0;
        r.check(nx_optimizer_size(r.opt, g, &count));
        std::vector<double> v(static_cast<size_t>(count));
        r.check(nx_optimizer_download(r.ctx, r.opt, r.scene, g, v.data(), nullptr, nullptr));
        if (g < 7) {
            const int c0 = kGroupCols[g][0], w = kGroupCols[g][1];
            for (size_t i = 0; i < n; ++i) {
                double* p = &s.nexels[i].mu.x;
                for (int k = 0; k < w; ++k) p[c0 + k] = v[i * w + k];
            }
        } else {
            std::vector<double>* dst[4] = {&s.field.grid.table, &s.field.mlp.w1, &s.field.mlp.w2, &s.field.mlp.w3};
            *dst[g - 7] = std::move(v);
        }
    }
    return s;
}

// mean_psnr (trainer.cpp:215-229) on the device scene: clamp01 renders vs the images.
double device_mean_psnr(const Run& r, const Bundle& bundle, const std::vector<int>& views, void* stream) {
    if (views.empty()) return 0.0;
    double acc = 0.0;
    for (int v : views) {
        const nx_camera cam = to_nx(bundle.cameras[v]);
        r.check(nx_render(r.ctx, r.scene, &cam, r.frame, stream));
        const size_t npix = static_cast<size_t>(cam.width) * cam.height;
        std::vector<float> fin(npix * 3);
        nx_host_frame h{};
        h.final_img = fin.data();
        r.check(nx_frame_download(r.ctx, r.frame, &h, stream));
        r.check(nx_ctx_synchronize(r.ctx));
        Image img;
        img.width = cam.width;
        img.height = cam.height;
        img.px.resize(npix * 3);
        for (size_t i = 0; i < img.px.size(); ++i) img.px[i] = std::min(1.0, std::max(0.0, static_cast<double>(fin[i])));
        acc += psnr(img, bundle.images[v]);
    }
    return acc / static_cast<double>(views.size());
}

}  // namespace

// mean_psnr (trainer.cpp:215-229) over the GPU-backed render (host/renderer_b200.cpp).
double mean_psnr(const Scene& scene, const Bundle& bundle, const std::vector<int>& views) {
    if (views.empty()) return 0.0;
    double acc = 0.0;
    for (int v : views) {
        const RenderResult res = render(scene, bundle.cameras[v]);
        Image img;
        img.width = bundle.images[v].width;
        img.height = bundle.images[v].height;
        img.px = res.fb.final_img;
        for (double& x : img.px) x = std::min(1.0, std::max(0.0, x));
        acc += psnr(img, bundle.images[v]);
    }
    return acc / static_cast<double>(views.size());
}

TrainResult train(const Bundle& bundle, const TrainConfig& cfg, const TrainHooks& hooks) {
    if (bundle.train_views.empty()) fail("bad-settings", "bundle has no train views");
    if (cfg.iterations < 0) fail("bad-config", "iterations must be >= 0");
    if (cfg.top_k < 0 || cfg.top_k > kMaxTopK)
        fail("bad-config", "top_k must be in [0, " + std::to_string(kMaxTopK) + "]");

    std::mt19937_64 rng(cfg.seed);
    TrainResult out;
    out.scene = initialize_scene(bundle, cfg, rng);
    const Scene init = out.scene;
    out.extra.cameras = bundle.cameras;
    out.optimizer.assign(kGroupCount, AdamState{});

    nx_adam_config gcfg[kGroupCount];
    const double ext = init.extent;
    const double lrs[kGroupCount] = {cfg.lr_position * ext, cfg.lr_quat, cfg.lr_scale, cfg.lr_opacity, cfg.lr_gamma,
                                     cfg.lr_sh_dc, cfg.lr_sh_rest, cfg.lr_grid, cfg.lr_mlp, cfg.lr_mlp, cfg.lr_mlp};
    for (int g = 0; g < kGroupCount; ++g)
        gcfg[g] = nx_adam_config{lrs[g], 0.9, 0.999, g == kGroupPosition ? cfg.adam_eps_position : cfg.adam_eps};
    const double decay = cfg.lr_position_final / std::max(cfg.lr_position, std::numeric_limits<double>::min());

    // ---- device run state
    Run r;
    const char* env = std::getenv("NEXEL_CUDA_DEVICE");
    int device = env ? std::atoi(env) : 0;
    const int dp_world = dp_env_world(), dp_rank = dp_env_rank();
    if (!env && dp_world > 1) {  // one GPU per rank unless the device is given
        int count = 1;
        cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        device = dp_rank % std::max(count, 1);
    }
    r.check(nx_ctx_create(device, &r.ctx));
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    const std::unique_ptr<DpComm> dp = DpComm::from_env(device);
    void* s = nx_ctx_stream(r.ctx);
    cudaStream_t cs = static_cast<cudaStream_t>(s);
    const nx_settings st = to_nx(init.settings);
    const auto& gc = init.field.grid.cfg;
    const nx_field_desc fd{gc.levels, gc.log2_table, gc.features, init.field.mlp.n_hidden, gc.base_scale, gc.growth};
    r.check(nx_scene_create(r.ctx, &st, static_cast<int64_t>(init.nexels.size()),
                            init.nexels.empty() ? nullptr : &init.nexels[0].mu.x, &fd, init.field.grid.table.data(),
                            init.field.mlp.w1.data(), init.field.mlp.w2.data(), init.field.mlp.w3.data(), &r.scene));
    r.check(nx_frame_create(r.ctx, 0, 0, 0, &r.frame));
    r.check(nx_frame_set_backward(r.ctx, r.frame, 1));
    r.check(nx_optimizer_create(r.ctx, r.scene, &r.opt));
    for (int g = kGroupShDc; g < kGroupCount; ++g) {  // exact fp64 masters of the fp32-stored groups
        const std::vector<double> rows = group_rows(init, g);
        r.check(nx_optimizer_set_params(r.ctx, r.opt, r.scene, g, rows.data(), static_cast<int64_t>(rows.size())));
    }

    DevArena mem;
    int max_pix = 0;
    std::vector<double*> gt(bundle.cameras.size(), nullptr);  // train views' ground truth, resident
    for (int v : bundle.train_views) {
        if (gt[v]) continue;
        const Image& im = bundle.images[v];
        const size_t npx = static_cast<size_t>(im.width) * im.height;
        if (bundle.cameras[v].width != im.width || bundle.cameras[v].height != im.height || im.px.size() != npx * 3)
            fail("bad-settings", "train view " + std::to_string(v) + ": image does not match its camera");
        gt[v] = mem.alloc<double>(npx * 3);
        cuda_check(cudaMemcpyAsync(gt[v], im.px.data(), npx * 3 * sizeof(double), cudaMemcpyHostToDevice, cs),
                   "gt upload");
        max_pix = std::max<int>(max_pix, static_cast<int>(npx));
    }
    const int K = init.settings.top_k;
    double* d_final = mem.alloc<double>(static_cast<size_t>(max_pix) * 3);
    double* d_weights = mem.alloc<double>(static_cast<size_t>(max_pix) * std::max(K, 1));
    double* d_texture = mem.alloc<double>(static_cast<size_t>(max_pix) * std::max(K, 1) * 3);
    double* err_pixel = mem.alloc<double>(static_cast<size_t>(max_pix));
    nx_loss_terms* d_terms = mem.alloc<nx_loss_terms>(1);
    const size_t n_table = init.field.grid.table.size(), n_w1 = init.field.mlp.w1.size(),
                 n_w2 = init.field.mlp.w2.size(), n_w3 = init.field.mlp.w3.size();
    double* g_table = mem.alloc<double>(n_table);
    double* g_w1 = mem.alloc<double>(n_w1);
    double* g_w2 = mem.alloc<double>(n_w2);
    double* g_w3 = mem.alloc<double>(n_w3);
    size_t n = init.nexels.size(), cap = std::max<size_t>(n, 1);
    double* g_prims = mem.alloc<double>(cap * NX_PARAMS_PER_NEXEL);
    double* err_accum = mem.alloc<double>(cap);
    cuda_check(cudaMemsetAsync(err_accum, 0, cap * sizeof(double), cs), "memset");
    double* uniforms = nullptr;
    size_t ucap = 0;

    std::vector<int> perm;
    size_t perm_pos = 0;
    LossTerms terms;
    // NEXEL_TRAIN_PROFILE=1: per-phase wall times (synchronising after each phase) on stderr
    static const bool profile = std::getenv("NEXEL_TRAIN_PROFILE") != nullptr;
    double phase_s[6] = {};
    auto tp = std::chrono::steady_clock::now();
    auto mark = [&](int phase) {
        if (!profile) return;
        cuda_check(cudaStreamSynchronize(cs), "sync");
        const auto now = std::chrono::steady_clock::now();
        phase_s[phase] += std::chrono::duration<double>(now - tp).count();
        tp = now;
    };
    for (int iter = 1; iter <= cfg.iterations; ++iter) {
        const auto t0 = std::chrono::steady_clock::now();
        tp = t0;
        int view = -1;
        for (int q = 0; q < dp_world; ++q) {  // this rank's position of the iteration's dp_world
            if (perm_pos == perm.size()) {    // trainer.cpp:280-284
                perm = bundle.train_views;
                std::shuffle(perm.begin(), perm.end(), rng);
                perm_pos = 0;
            }
            const int v = perm[perm_pos++];
            if (q == dp_rank) view = v;
        }
        const nx_camera cam = to_nx(bundle.cameras[view]);
        const size_t npix = static_cast<size_t>(cam.width) * cam.height;

        r.check(nx_render(r.ctx, r.scene, &cam, r.frame, s));
        mark(0);
        cuda_check(cudaMemsetAsync(g_prims, 0, n * NX_PARAMS_PER_NEXEL * sizeof(double), cs), "memset");
        cuda_check(cudaMemsetAsync(g_table, 0, n_table * sizeof(double), cs), "memset");
        cuda_check(cudaMemsetAsync(g_w1, 0, n_w1 * sizeof(double), cs), "memset");
        cuda_check(cudaMemsetAsync(g_w2, 0, n_w2 * sizeof(double), cs), "memset");
        cuda_check(cudaMemsetAsync(g_w3, 0, n_w3 * sizeof(double), cs), "memset");
        const nx_grads grads{g_prims, g_table, g_w1, g_w2, g_w3};
        const nx_loss_weights lw{cfg.loss.dssim, cfg.loss.alpha, cfg.loss.texture, cfg.loss.opacity, cfg.loss.grid};
        r.check(nx_losses_backward_opt(r.ctx, r.scene, r.frame, gt[view], &lw, d_final, K ? d_weights : nullptr,
                                       K ? d_texture : nullptr, &grads, d_terms, r.opt, s));
        static_assert(sizeof(nx_loss_terms) == 8 * sizeof(double), "loss terms: 8 doubles");
        if (dp) dp->all_reduce(reinterpret_cast<double*>(d_terms), 8, true, cs);  // the ranks' mean loss
        nx_loss_terms ht;
        cuda_check(cudaMemcpyAsync(&ht, d_terms, sizeof ht, cudaMemcpyDeviceToHost, cs), "terms");
        cuda_check(cudaStreamSynchronize(cs), "sync");
        terms = from_nx(ht);
        if (!terms.finite()) {  // trainer.cpp:291-299
            if (!cfg.snapshot_path.empty() && dp_rank == 0) {
                CheckpointExtra snap;
                snap.cameras = bundle.cameras;
                snap.iteration = static_cast<std::uint64_t>(iter);
                save_checkpoint(cfg.snapshot_path, download_scene(r, init), snap);
            }
            fail("non-finite-loss", "loss diverged at iteration " + std::to_string(iter));
        }
        (void)npix;
        mark(1);
        r.check(nx_pixel_error(r.ctx, r.frame, gt[view], err_pixel, s));
        const nx_upstream up{d_final, K ? d_weights : nullptr, K ? d_texture : nullptr};
        r.check(nx_render_backward(r.ctx, r.scene, &cam, r.frame, &up, &grads, err_pixel, err_accum, s));
        if (dp) {  // the replicas' mean gradient (in place, on the run's stream)
            dp->all_reduce(g_prims, n * NX_PARAMS_PER_NEXEL, true, cs);
            dp->all_reduce(g_table, n_table, true, cs);
            dp->all_reduce(g_w1, n_w1, true, cs);
            dp->all_reduce(g_w2, n_w2, true, cs);
            dp->all_reduce(g_w3, n_w3, true, cs);
        }
        mark(2);

        gcfg[kGroupPosition].lr = cfg.lr_position * ext *
                                  std::pow(decay, static_cast<double>(iter) / std::max(1, cfg.iterations));
        r.check(nx_optimizer_step(r.ctx, r.opt, r.scene, &grads, gcfg, s));
        mark(3);

        if (cfg.densify_every > 0 && iter % cfg.densify_every == 0 && iter >= cfg.densify_start &&
            iter <= cfg.densify_end) {  // trainer.cpp:324-333
            if (dp) dp->all_reduce(err_accum, n, false, cs);  // every rank's views' blended errors
            cuda_check(cudaStreamSynchronize(cs), "sync");
            const int allowed = std::min(static_cast<int>(std::ceil(cfg.split_fraction * static_cast<double>(n))),
                                         cfg.budget - static_cast<int>(n));
            int64_t n_out = static_cast<int64_t>(n), splits = 0;
            if (n > 0 && allowed > 0) {  // density.cpp:103-121: one draw per nexel, in order
                std::vector<double> u(n);
                std::uniform_real_distribution<double> uni(0.0, 1.0);
                for (size_t i = 0; i < n; ++i) u[i] = uni(rng);
                if (n > ucap) {
                    if (uniforms) mem.release(uniforms);
                    ucap = n;
                    uniforms = mem.alloc<double>(ucap);
                }
                cuda_check(cudaMemcpyAsync(uniforms, u.data(), n * sizeof(double), cudaMemcpyHostToDevice, cs),
                           "uniforms");
                r.check(nx_scene_densify_split(r.ctx, r.scene, r.opt, err_accum, uniforms, cfg.budget,
                                               cfg.split_fraction, nullptr, &n_out, &splits));
            }
            r.check(nx_scene_prune(r.ctx, r.scene, r.opt, cfg.prune_opacity, nullptr, &n_out));
            n = static_cast<size_t>(n_out);
            if (n > cap) {
                mem.release(g_prims);
                mem.release(err_accum);
                cap = n;
                g_prims = mem.alloc<double>(cap * NX_PARAMS_PER_NEXEL);
                err_accum = mem.alloc<double>(cap);
            }
            cuda_check(cudaMemsetAsync(err_accum, 0, std::max<size_t>(n, 1) * sizeof(double), cs), "memset");
        }

        mark(4);
        cuda_check(cudaStreamSynchronize(cs), "sync");
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.last_loss = terms;
        if (hooks.on_iteration) hooks.on_iteration(iter, terms, static_cast<int>(n), wall);
        if (hooks.on_eval && cfg.eval_every > 0 && (iter % cfg.eval_every == 0 || iter == cfg.iterations))
            hooks.on_eval(iter, device_mean_psnr(r, bundle, bundle.train_views, s),
                          device_mean_psnr(r, bundle, bundle.test_views, s));
    }

    if (profile && cfg.iterations > 0) {
        const char* names[5] = {"render", "losses", "backward", "adam", "density"};
        for (int p = 0; p < 5; ++p)
            std::fprintf(stderr, "train profile: %-8s %.3f ms/iteration\n", names[p], 1e3 * phase_s[p] / cfg.iterations);
    }
    // ---- results: fp64 parameters and Adam states (trainer.cpp:346-348)
    out.scene = download_scene(r, init);
    int64_t steps[NX_NUM_GROUPS];
    r.check(nx_optimizer_steps(r.opt, steps));
    for (int g = 0; g < kGroupCount; ++g) {
        AdamState& a = out.optimizer[g];
        a.step = steps[g];
        if (a.step == 0) continue;  // adam_step sizes the moments on first use
        int64_t count = 0;
        r.check(nx_optimizer_size(r.opt, g, &count));
        a.m.resize(static_cast<size_t>(count));
        a.v.resize(static_cast<size_t>(count));
        r.check(nx_optimizer_download(r.ctx, r.opt, r.scene, g, nullptr, a.m.data(), a.v.data()));
    }
    out.extra.iteration = static_cast<std::uint64_t>(cfg.iterations);
    return out;
}

}  // namespace nexel
