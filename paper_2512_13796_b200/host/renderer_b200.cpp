// Drop-in replacement for the render path of proj/core/src/renderer.cpp:
// nexel::validate_settings, collection_pass, texturing_pass, render and
// render_backward with the reference's signatures (include/nexel/renderer.hpp:22-53,
// scene.hpp:35), running on the sm_100a library through its C-ABI
// (include/nexel_b200.h).
//
// Compiled against the reference's public headers and linked in place of
// renderer.cpp's forward half. Semantics kept:
//   * validation order and codes: bad-settings, then bad-camera (the reference's
//     own validate_camera), then bad-primitive with the first failing id;
//   * FrameBuffers::allocate shapes and sentinels, RenderResult::blended_error zeroed;
//   * collection_pass and texturing_pass separately callable; texturing_pass
//     consumes the host FrameBuffers it is given (uploaded if they are not the ones
//     the device frame holds).
// The device scene is cached per Scene content (fingerprint of every parameter).
#include "nexel/renderer.hpp"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nexel/error.hpp"
#include "../../include/nexel_b200.h"

namespace nexel {

namespace {

struct Device {
    nx_ctx* ctx = nullptr;
    nx_scene* scene = nullptr;
    nx_frame* frame = nullptr;
    uint64_t scene_key = 0;
    const FrameBuffers* frame_owner = nullptr;  // host FrameBuffers mirrored by `frame`
    std::mutex mu;
};

Device& device() {
    static Device d;
    return d;
}

[[noreturn]] void raise(int status, const std::string& msg) {
    const char* code = nx_status_name(status);
    fail(code, msg);
}

void check(Device& d, int status) {
    if (status == NX_OK) return;
    int st = status;
    const char* msg = d.ctx ? nx_ctx_last_error(d.ctx, &st) : "no CUDA context";
    raise(status, msg);
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

uint64_t fingerprint(const Scene& s) {
    uint64_t h = 1469598103934665603ull;
    h = fnv(h, s.nexels.data(), s.nexels.size() * sizeof(Nexel));
    h = fnv(h, s.field.grid.table.data(), s.field.grid.table.size() * sizeof(double));
    for (const auto* w : {&s.field.mlp.w1, &s.field.mlp.w2, &s.field.mlp.w3})
        h = fnv(h, w->data(), w->size() * sizeof(double));
    const int shape[5] = {s.field.grid.cfg.levels, s.field.grid.cfg.log2_table, s.field.grid.cfg.features,
                          s.field.mlp.n_hidden, static_cast<int>(s.nexels.size())};
    h = fnv(h, shape, sizeof shape);
    h = fnv(h, &s.field.grid.cfg.base_scale, sizeof(double));
    h = fnv(h, &s.field.grid.cfg.growth, sizeof(double));
    return h;
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

// Context + device scene for `scene` (uploaded when its content changed).
Device& bind(const Scene& scene) {
    Device& d = device();
    if (!d.ctx) {
        const char* env = std::getenv("NEXEL_CUDA_DEVICE");
        const int dev = env ? std::atoi(env) : 0;
        const int st = nx_ctx_create(dev, &d.ctx);
        if (st != NX_OK) raise(st, "cannot create a CUDA context on device " + std::to_string(dev));
        check(d, nx_frame_create(d.ctx, 0, 0, 0, &d.frame));
        check(d, nx_frame_set_backward(d.ctx, d.frame, 1));  // fp64 base, as FrameBuffers holds it
    }
    const uint64_t key = fingerprint(scene);
    const nx_settings st = to_nx(scene.settings);
    if (!d.scene || key != d.scene_key) {
        if (d.scene) nx_scene_destroy(d.scene);
        d.scene = nullptr;
        const auto& g = scene.field.grid.cfg;
        nx_field_desc fd{g.levels, g.log2_table, g.features, scene.field.mlp.n_hidden, g.base_scale, g.growth};
        const double* nex = scene.nexels.empty() ? nullptr : &scene.nexels[0].mu.x;
        check(d, nx_scene_create(d.ctx, &st, static_cast<int64_t>(scene.nexels.size()), nex, &fd,
                                 scene.field.grid.table.data(), scene.field.mlp.w1.data(),
                                 scene.field.mlp.w2.data(), scene.field.mlp.w3.data(), &d.scene));
        d.scene_key = key;
    }
    check(d, nx_scene_set_settings(d.ctx, d.scene, &st));
    return d;
}

template <typename T>
void widen(const std::vector<T>& src, std::vector<double>& dst) {
    dst.resize(src.size());
    for (size_t i = 0; i < src.size(); ++i) dst[i] = static_cast<double>(src[i]);
}

}  // namespace

// validate_settings (renderer.cpp:13-21): identical checks and messages.
void validate_settings(const RenderSettings& s) {
    if (s.top_k < 0 || s.top_k > kMaxTopK)
        fail("bad-settings", "top_k must be in [0, " + std::to_string(kMaxTopK) + "], got " + std::to_string(s.top_k));
    if (!(s.near_eps > 0)) fail("bad-settings", "near_eps must be positive");
    if (!(s.alpha_max > 0) || s.alpha_max >= 1) fail("bad-settings", "alpha_max must be in (0,1)");
    if (!(s.min_transmittance >= 0)) fail("bad-settings", "min_transmittance must be >= 0");
    if (s.tile < 1) fail("bad-settings", "tile must be >= 1");
}

void collection_pass(const Scene& scene, const Camera& cam, RenderResult& out) {
    validate_settings(scene.settings);
    validate_camera(cam);  // the reference's own (camera.cpp:8-31): same messages
    const int K = scene.settings.top_k;
    out.fb.allocate(cam.width, cam.height, K);
    out.blended_error.assign(scene.nexels.size(), 0.0);
    Device& d = bind(scene);
    std::lock_guard<std::mutex> lock(d.mu);
    const nx_camera c = to_nx(cam);
    check(d, nx_collection_pass(d.ctx, d.scene, &c, d.frame, nullptr));
    nx_host_frame h{};
    h.base_f64 = out.fb.base.data();          // the fp64 base (Eq. 6) the device kept
    h.residual_f64 = out.fb.residual.data();  // and the fp64 terminal transmittance
    h.ids = out.fb.ids.data();
    h.depths = out.fb.depths.data();
    h.weights = out.fb.weights.data();
    check(d, nx_frame_download(d.ctx, d.frame, &h, nullptr));
    check(d, nx_ctx_synchronize(d.ctx));
    d.frame_owner = &out.fb;
}

void texturing_pass(const Scene& scene, const Camera& cam, FrameBuffers& fb) {
    if (fb.top_k == 0) {  // renderer.cpp:208-211
        fb.final_img = fb.base;
        return;
    }
    Device& d = bind(scene);
    std::lock_guard<std::mutex> lock(d.mu);
    const size_t npix = static_cast<size_t>(fb.width) * fb.height;
    if (d.frame_owner != &fb) {  // not the frame collection_pass just produced: upload it
        std::vector<float> base(fb.base.begin(), fb.base.end());
        nx_host_frame h{};
        h.base = base.data();
        h.ids = fb.ids.data();
        h.depths = fb.depths.data();
        h.weights = fb.weights.data();
        check(d, nx_frame_upload(d.ctx, d.frame, fb.width, fb.height, fb.top_k, &h, nullptr));
    }
    const nx_camera c = to_nx(cam);
    check(d, nx_texturing_pass(d.ctx, d.scene, &c, d.frame, nullptr));
    std::vector<float> texture(npix * fb.top_k * 3), final_img(npix * 3);
    nx_host_frame h{};
    h.texture = texture.data();
    h.final_img = final_img.data();
    check(d, nx_frame_download(d.ctx, d.frame, &h, nullptr));
    check(d, nx_ctx_synchronize(d.ctx));
    widen(texture, fb.texture);
    widen(final_img, fb.final_img);
}

RenderResult render(const Scene& scene, const Camera& cam) {  // renderer.cpp:239-244
    RenderResult out;
    collection_pass(scene, cam, out);
    texturing_pass(scene, cam, out.fb);
    return out;
}

// render_backward (renderer.hpp:50-53, renderer.cpp:251-401): the host FrameBuffers
// (the forward's output) are uploaded, the reverse pass runs on the device and the
// gradients are accumulated into `grads` / `blended_error` like the reference.
void render_backward(const Scene& scene, const Camera& cam, const FrameBuffers& fb, const UpstreamGrads& up,
                     SceneGrads& grads, const double* err_pixel, std::vector<double>* blended_error) {
    validate_settings(scene.settings);
    validate_camera(cam);
    if (grads.prims.size() != scene.nexels.size() || grads.field.table.size() != scene.field.grid.table.size() ||
        grads.field.w1.size() != scene.field.mlp.w1.size() || grads.field.w2.size() != scene.field.mlp.w2.size() ||
        grads.field.w3.size() != scene.field.mlp.w3.size())
        fail("invalid-argument", "render_backward: SceneGrads not allocated for this scene");
    if (blended_error && blended_error->size() != scene.nexels.size())
        fail("invalid-argument", "render_backward: blended_error does not match the scene");
    Device& d = bind(scene);
    std::lock_guard<std::mutex> lock(d.mu);
    const size_t npix = static_cast<size_t>(fb.width) * fb.height;
    std::vector<float> texture(fb.texture.begin(), fb.texture.end());
    std::vector<float> base32(fb.base.begin(), fb.base.end()), residual(fb.residual.begin(), fb.residual.end());
    nx_host_frame h{};
    h.base = base32.data();
    h.base_f64 = const_cast<double*>(fb.base.data());
    h.ids = const_cast<int32_t*>(fb.ids.data());
    h.depths = const_cast<double*>(fb.depths.data());
    h.weights = const_cast<double*>(fb.weights.data());
    h.texture = texture.data();
    h.residual = residual.data();
    h.residual_f64 = const_cast<double*>(fb.residual.data());
    (void)npix;
    check(d, nx_frame_upload(d.ctx, d.frame, fb.width, fb.height, fb.top_k, &h, nullptr));
    d.frame_owner = nullptr;
    static_assert(sizeof(PrimitiveGrad) == NX_PARAMS_PER_NEXEL * sizeof(double), "PrimitiveGrad = 60 doubles");
    nx_grads g{grads.prims.empty() ? nullptr : &grads.prims[0].mu.x, grads.field.table.data(), grads.field.w1.data(),
               grads.field.w2.data(), grads.field.w3.data()};
    const bool k = fb.top_k > 0;
    nx_upstream u{up.d_final, k ? up.d_weights : nullptr, k ? up.d_texture : nullptr};
    const nx_camera c = to_nx(cam);
    check(d, nx_render_backward_host(d.ctx, d.scene, &c, d.frame, &u, &g, err_pixel,
                                     blended_error ? blended_error->data() : nullptr));
}

}  // namespace nexel
