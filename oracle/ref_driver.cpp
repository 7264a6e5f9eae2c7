// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// C-ABI over the *reference* renderer, compiled in place from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/ (git-ignored).
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load it,
// and only as the checker / CPU timing baseline.
//
// This translation unit #includes the reference's renderer.cpp so that the
// anonymous-namespace Binning / build_binning (renderer.cpp:25-111) are
// reachable for key-level parity; renderer.cpp is therefore
// not linked separately. The reference's own test helpers (tests/helpers.hpp)
// provide the seeded scene/camera generators (random_nexel, init_field,
// orbit_camera, look_at_camera), whose outputs depend on libstdc++ and are
// therefore generated here rather than re-implemented.
#include "renderer.cpp"  // -I /root/reference/proj/core/src: compiled in place, not copied
#include "helpers.hpp"                                  // -I /root/reference/proj/tests

#include "nexel/adam.hpp"
#include "nexel/checkpoint.hpp"
#include "nexel/density.hpp"
#include "nexel/losses.hpp"
#include "nexel/oracle.hpp"

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

#include "../include/nexel_b200.h"

using namespace nexel;

namespace {

thread_local std::string g_err;

int status_of(const Error& e) {
    if (e.code() == "bad-settings") return NX_BAD_SETTINGS;
    if (e.code() == "bad-camera") return NX_BAD_CAMERA;
    if (e.code() == "bad-primitive") return NX_BAD_PRIMITIVE;
    return NX_INVALID_ARGUMENT;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return NX_OK;
    } catch (const Error& e) {
        g_err = e.code() + ": " + e.what();
        return status_of(e);
    } catch (const std::exception& e) {
        g_err = std::string("exception: ") + e.what();
        return NX_INVALID_ARGUMENT;
    }
}

RenderSettings to_settings(const nx_settings& s) {
    RenderSettings r;
    r.top_k = s.top_k;
    r.tile = s.tile;
    r.background = {s.background[0], s.background[1], s.background[2]};
    r.near_eps = s.near_eps;
    r.alpha_max = s.alpha_max;
    r.min_transmittance = s.min_transmittance;
    r.no_gamma = s.no_gamma != 0;
    r.no_prim_sh = s.no_prim_sh != 0;
    r.no_downweight = s.no_downweight != 0;
    return r;
}

nx_settings from_settings(const RenderSettings& r) {
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

Camera to_camera(const nx_camera& c) {
    Camera cam;
    cam.name = "nx";
    cam.width = c.width;
    cam.height = c.height;
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) cam.R.m[r][k] = c.R[r * 3 + k];
        cam.t[r] = c.t[r];
    }
    return cam;
}

nx_camera from_camera(const Camera& cam) {
    nx_camera c;
    std::memset(&c, 0, sizeof c);
    c.width = cam.width;
    c.height = cam.height;
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) c.R[r * 3 + k] = cam.R.m[r][k];
        c.t[r] = cam.t[r];
    }
    return c;
}

void export_scene(const Scene& s, double* nexels, nx_settings* settings, nx_field_desc* field,
                  double* table, double* w1, double* w2, double* w3) {
    if (nexels)
        for (std::size_t i = 0; i < s.nexels.size(); ++i)
            std::memcpy(nexels + i * NX_PARAMS_PER_NEXEL, &s.nexels[i], sizeof(Nexel));
    if (settings) *settings = from_settings(s.settings);
    if (field) {
        field->levels = s.field.grid.cfg.levels;
        field->log2_table = s.field.grid.cfg.log2_table;
        field->features = s.field.grid.cfg.features;
        field->n_hidden = s.field.mlp.n_hidden;
        field->base_scale = s.field.grid.cfg.base_scale;
        field->growth = s.field.grid.cfg.growth;
    }
    if (table) std::memcpy(table, s.field.grid.table.data(), s.field.grid.table.size() * 8);
    if (w1) std::memcpy(w1, s.field.mlp.w1.data(), s.field.mlp.w1.size() * 8);
    if (w2) std::memcpy(w2, s.field.mlp.w2.data(), s.field.mlp.w2.size() * 8);
    if (w3) std::memcpy(w3, s.field.mlp.w3.data(), s.field.mlp.w3.size() * 8);
}

static_assert(sizeof(Nexel) == NX_PARAMS_PER_NEXEL * sizeof(double), "Nexel is 60 packed doubles");

}  // namespace

struct ref_scene {
    Scene scene;
};

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_scene_create(const nx_settings* settings, int64_t n, const double* nexels,
                     const nx_field_desc* field, const double* table, const double* w1,
                     const double* w2, const double* w3, ref_scene** out) {
    return guarded([&] {
        auto h = std::make_unique<ref_scene>();
        Scene& s = h->scene;
        s.settings = to_settings(*settings);
        s.nexels.resize(static_cast<std::size_t>(n));
        if (n) std::memcpy(s.nexels.data(), nexels, static_cast<std::size_t>(n) * sizeof(Nexel));
        HashGridConfig cfg;
        cfg.levels = field->levels;
        cfg.log2_table = field->log2_table;
        cfg.features = field->features;
        cfg.base_scale = field->base_scale;
        cfg.growth = field->growth;
        s.field.grid.cfg = cfg;
        s.field.grid.table.assign(table, table + cfg.param_count());
        s.field.mlp.n_in = cfg.levels * cfg.features;
        s.field.mlp.n_hidden = field->n_hidden;
        s.field.mlp.n_out = NX_SH_VALUES;
        s.field.mlp.allocate();
        std::memcpy(s.field.mlp.w1.data(), w1, s.field.mlp.w1.size() * 8);
        std::memcpy(s.field.mlp.w2.data(), w2, s.field.mlp.w2.size() * 8);
        std::memcpy(s.field.mlp.w3.data(), w3, s.field.mlp.w3.size() * 8);
        *out = h.release();
    });
}

void ref_scene_destroy(ref_scene* h) { delete h; }

int ref_scene_set_settings(ref_scene* h, const nx_settings* settings) {
    h->scene.settings = to_settings(*settings);
    return NX_OK;
}

// nexel::render (renderer.cpp:239-244); any output pointer may be NULL.
int ref_render(const ref_scene* h, const nx_camera* c, double* base, int32_t* ids, double* depths,
               double* weights, double* texture, double* final_img, double* residual) {
    return guarded([&] {
        const RenderResult rr = render(h->scene, to_camera(*c));
        const FrameBuffers& fb = rr.fb;
        auto put = [](auto* dst, const auto& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
        };
        put(base, fb.base);
        put(ids, fb.ids);
        put(depths, fb.depths);
        put(weights, fb.weights);
        put(texture, fb.texture);
        put(final_img, fb.final_img);
        put(residual, fb.residual);
    });
}

// nexel::naive_render (oracle.cpp:13-90): rgb H*W*3.
int ref_naive_render(const ref_scene* h, const nx_camera* c, double* img) {
    return guarded([&] {
        const Image im = naive_render(h->scene, to_camera(*c));
        std::memcpy(img, im.px.data(), im.px.size() * 8);
    });
}

// Binning::tile_lists from build_binning (renderer.cpp:36-111).
int ref_tile_lists(const ref_scene* h, const nx_camera* c, int64_t* offsets, int32_t* ids,
                   int64_t capacity, int64_t* total, int32_t* tiles_x, int32_t* tiles_y) {
    return guarded([&] {
        validate_settings(h->scene.settings);
        const Camera cam = to_camera(*c);
        validate_camera(cam);
        const Binning bin = build_binning(h->scene, cam);
        *tiles_x = bin.tiles_x;
        *tiles_y = bin.tiles_y;
        int64_t at = 0;
        for (std::size_t t = 0; t < bin.tile_lists.size(); ++t) {
            if (offsets) offsets[t] = at;
            for (std::int32_t id : bin.tile_lists[t]) {
                if (ids && at < capacity) ids[at] = id;
                ++at;
            }
        }
        if (offsets) offsets[bin.tile_lists.size()] = at;
        *total = at;
    });
}

// Per-pixel contributor sequences: the exact march of collection_pass
// (renderer.cpp:137-153) with the reference's own intersect(), recording ids.
int ref_pixel_hits(const ref_scene* h, const nx_camera* c, int y0, int y1, int max_hits,
                   int32_t* hits, int32_t* counts) {
    return guarded([&] {
        const Scene& scene = h->scene;
        const RenderSettings& st = scene.settings;
        validate_settings(st);
        const Camera cam = to_camera(*c);
        validate_camera(cam);
        const Binning bin = build_binning(scene, cam);
        const int tile = st.tile;
        const int W = cam.width;
        const int rows = y1 - y0;
        parallel_chunks(static_cast<std::size_t>(rows) * W, 256,
                        [&](std::size_t, std::size_t b, std::size_t e) {
            for (std::size_t q = b; q < e; ++q) {
                const int py = y0 + static_cast<int>(q / W);
                const int px = static_cast<int>(q % W);
                const auto& list = bin.tile_lists[static_cast<std::size_t>(py / tile) * bin.tiles_x +
                                                  px / tile];
                const Ray ray = cam.pixel_ray(px + 0.5, py + 0.5);
                double T = 1.0;
                int n = 0;
                for (std::int32_t id : list) {
                    const SurfelHit hh = intersect(bin.act[id], ray, st.near_eps);
                    if (!hh.hit) continue;
                    if (n < max_hits) hits[q * max_hits + n] = id;
                    ++n;
                    const double alpha = std::min(hh.alpha, st.alpha_max);
                    T *= 1.0 - alpha;
                    if (T < st.min_transmittance) break;
                }
                counts[q] = n;
            }
        });
    });
}

// Seeded scene + orbit camera with the reference test generators
// (tests/helpers.hpp:88-125): g(seed); background; n x random_nexel; init_field;
// orbit_camera. Sizes follow from the arguments (see field desc).
int ref_gen_random_scene(uint64_t seed, int n_prims, int top_k, double op_lo, double op_hi,
                         int levels, int log2_table, double grid_init, int hidden, int res,
                         double focal, double dist, double* nexels, nx_settings* settings,
                         nx_field_desc* field, double* table, double* w1, double* w2, double* w3,
                         nx_camera* cam) {
    return guarded([&] {
        std::mt19937_64 g(seed);
        Scene scene;
        scene.settings.top_k = top_k;
        scene.settings.background = {testutil::urand(g, 0, 1), testutil::urand(g, 0, 1),
                                     testutil::urand(g, 0, 1)};
        for (int i = 0; i < n_prims; ++i)
            scene.nexels.push_back(testutil::random_nexel(g, 0.6, 0.15, 0.45, op_lo, op_hi));
        testutil::init_field(scene.field, g, levels, log2_table, grid_init, hidden);
        const Camera c = testutil::orbit_camera(g, res, focal, dist);
        export_scene(scene, nexels, settings, field, table, w1, w2, w3);
        *cam = from_camera(c);
    });
}

// init_field(field, g(seed), levels, log2, grid_init, hidden) alone (helpers.hpp:110-114).
int ref_gen_field(uint64_t seed, int levels, int log2_table, double grid_init, int hidden,
                  nx_field_desc* field, double* table, double* w1, double* w2, double* w3) {
    return guarded([&] {
        std::mt19937_64 g(seed);
        Scene scene;
        testutil::init_field(scene.field, g, levels, log2_table, grid_init, hidden);
        export_scene(scene, nullptr, nullptr, field, table, w1, w2, w3);
    });
}

// TextureField::init with HashGridConfig::for_extent (the stump_like field).
int ref_gen_field_for_extent(uint64_t seed, double extent, int levels, int log2_table,
                             double grid_init, nx_field_desc* field, double* table, double* w1,
                             double* w2, double* w3) {
    return guarded([&] {
        std::mt19937_64 g(seed);
        Scene scene;
        scene.field.init(HashGridConfig::for_extent(extent, levels, log2_table, 2), g, grid_init);
        export_scene(scene, nullptr, nullptr, field, table, w1, w2, w3);
    });
}

// look_at_camera (helpers.hpp:68-86).
int ref_look_at_camera(const double* pos, const double* target, int res, double focal,
                       nx_camera* cam) {
    return guarded([&] {
        *cam = from_camera(testutil::look_at_camera({pos[0], pos[1], pos[2]},
                                                    {target[0], target[1], target[2]}, res, focal));
    });
}

// Known-answer hooks for the geometry / field restatement tests.
double ref_eval_kernel(double u, double v, double o, double gx, double gy) {
    return eval_kernel(u, v, o, {gx, gy});
}
double ref_support_radius(double o, double g) { return support_radius(o, g); }
uint32_t ref_hash_cell(int64_t ix, int64_t iy, int64_t iz, uint32_t T) {
    return hash_cell(ix, iy, iz, T);
}
double ref_downweight(double s, double t, double f) { return downweight(s, t, f); }

// field_forward (texture_field.cpp:27-31) for a batch of (x, t, f, dir) queries.
int ref_field_forward(const ref_scene* h, int64_t n, const double* q8, int no_downweight,
                      double* rgb) {
    return guarded([&] {
        std::vector<FieldQuery> qs(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const double* r = q8 + i * 8;
            qs[i].x = {r[0], r[1], r[2]};
            qs[i].t = r[3];
            qs[i].f = r[4];
            qs[i].dir = {r[5], r[6], r[7]};
        }
        field_forward_batch(h->scene.field, qs, rgb, no_downweight != 0);
    });
}

// nexel::render + nexel::render_backward (renderer.cpp:239-401) with the given
// upstream gradients (any NULL = zero, renderer.hpp:40-44). Gradients of a fresh
// SceneGrads are written to g_* (PrimitiveGrad = 60 doubles per nexel in Nexel
// field order); blended_error (N, nullable) receives sum w * err_pixel.
int ref_render_backward(const ref_scene* h, const nx_camera* c, const double* d_final,
                        const double* d_weights, const double* d_texture, const double* err_pixel,
                        double* g_prims, double* g_table, double* g_w1, double* g_w2, double* g_w3,
                        double* blended_error) {
    return guarded([&] {
        const Scene& scene = h->scene;
        const Camera cam = to_camera(*c);
        RenderResult rr = render(scene, cam);
        SceneGrads grads;
        grads.allocate(scene);
        UpstreamGrads up;
        up.d_final = d_final;
        up.d_weights = d_weights;
        up.d_texture = d_texture;
        render_backward(scene, cam, rr.fb, up, grads, err_pixel,
                        blended_error ? &rr.blended_error : nullptr);
        static_assert(sizeof(PrimitiveGrad) == NX_PARAMS_PER_NEXEL * sizeof(double), "60 doubles");
        if (g_prims && !grads.prims.empty())
            std::memcpy(g_prims, grads.prims.data(), grads.prims.size() * sizeof(PrimitiveGrad));
        auto put = [](double* dst, const std::vector<double>& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
        };
        put(g_table, grads.field.table);
        put(g_w1, grads.field.w1);
        put(g_w2, grads.field.w2);
        put(g_w3, grads.field.w3);
        if (blended_error) put(blended_error, rr.blended_error);
    });
}

// nexel::losses_backward (losses.cpp:107-238) on a given FrameBuffers (ids, weights,
// texture, final_img: fp64 arrays as the reference holds them) and ground truth.
// lw = {dssim, alpha, texture, opacity, grid}; terms = {l1, dssim, image, texture,
// alpha, opacity, grid, total}. d_* are overwritten; g_prims (N*60) / g_table are
// accumulated into, as the reference does.
int ref_losses_backward(const ref_scene* h, int W, int H, int K, const int32_t* ids, const double* weights,
                        const double* texture, const double* final_img, const double* gt, const double* lw,
                        double* d_final, double* d_weights, double* d_texture, double* g_prims,
                        double* g_table, double* terms) {
    return guarded([&] {
        const Scene& scene = h->scene;
        FrameBuffers fb;
        fb.allocate(W, H, K);
        const size_t npix = static_cast<size_t>(W) * H;
        std::memcpy(fb.ids.data(), ids, npix * K * sizeof(int32_t));
        std::memcpy(fb.weights.data(), weights, npix * K * sizeof(double));
        std::memcpy(fb.texture.data(), texture, npix * K * 3 * sizeof(double));
        std::memcpy(fb.final_img.data(), final_img, npix * 3 * sizeof(double));
        Image img;
        img.allocate(W, H);
        std::memcpy(img.px.data(), gt, npix * 3 * sizeof(double));
        LossWeights w;
        w.dssim = lw[0];
        w.alpha = lw[1];
        w.texture = lw[2];
        w.opacity = lw[3];
        w.grid = lw[4];
        SceneGrads grads;
        grads.allocate(scene);
        std::memcpy(&grads.prims[0], g_prims, scene.nexels.size() * sizeof(PrimitiveGrad));
        std::memcpy(grads.field.table.data(), g_table, grads.field.table.size() * sizeof(double));
        std::vector<double> df, dw, dt;
        const LossTerms t = losses_backward(scene, fb, img, w, df, dw, dt, grads);
        std::memcpy(d_final, df.data(), df.size() * sizeof(double));
        if (K) {
            std::memcpy(d_weights, dw.data(), dw.size() * sizeof(double));
            std::memcpy(d_texture, dt.data(), dt.size() * sizeof(double));
        }
        std::memcpy(g_prims, &grads.prims[0], scene.nexels.size() * sizeof(PrimitiveGrad));
        std::memcpy(g_table, grads.field.table.data(), grads.field.table.size() * sizeof(double));
        const double tv[8] = {t.l1, t.dssim, t.image, t.texture, t.alpha, t.opacity, t.grid, t.total};
        std::memcpy(terms, tv, sizeof tv);
    });
}

// nexel::save_checkpoint (checkpoint.cpp:99-171) of the scene with the given cameras
// (named "cam<i>") and iteration counter; no optimizer section.
int ref_save_checkpoint(const ref_scene* h, const char* path, const nx_camera* cams, int n_cams,
                        uint64_t iteration, double extent) {
    return guarded([&] {
        Scene scene = h->scene;
        scene.extent = extent;
        CheckpointExtra extra;
        extra.iteration = iteration;
        for (int i = 0; i < n_cams; ++i) {
            Camera c = to_camera(cams[i]);
            c.name = "cam" + std::to_string(i);
            extra.cameras.push_back(c);
        }
        save_checkpoint(path, scene, extra);
    });
}

// nexel::adam_step (adam.cpp:9-22) on a flat block: m, v (count each) and *step are
// the AdamState, cfg = {lr, beta1, beta2, eps}; params updated in place.
int ref_adam_step(double* m, double* v, int64_t* step, const double* cfg, double* params, const double* grads,
                  int64_t count) {
    return guarded([&] {
        AdamState st;
        st.m.assign(m, m + count);
        st.v.assign(v, v + count);
        st.step = *step;
        AdamConfig c;
        c.lr = cfg[0];
        c.beta1 = cfg[1];
        c.beta2 = cfg[2];
        c.eps = cfg[3];
        adam_step(st, c, params, grads, static_cast<std::size_t>(count));
        std::memcpy(m, st.m.data(), count * sizeof(double));
        std::memcpy(v, st.v.data(), count * sizeof(double));
        *step = st.step;
    });
}

// nexel::densify_split (density.cpp:102-161) with std::mt19937_64(seed); nexels is
// N x 60 in / (N + splits) x 60 out (capacity cap rows); uniforms (N) receives the
// draws the call consumed (one per nexel, in order) for the device twin.
int ref_densify_split(double* nexels, int64_t n, int64_t cap, const double* errors, int64_t budget,
                      double split_fraction, uint64_t seed, double* uniforms, int32_t* new_to_old, int64_t* n_out,
                      int64_t* split_count) {
    return guarded([&] {
        std::vector<Nexel> nx(static_cast<size_t>(n));
        if (n) std::memcpy(nx.data(), nexels, n * sizeof(Nexel));
        std::vector<double> err(errors, errors + n);
        std::mt19937_64 draws(seed);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        for (int64_t i = 0; i < n; ++i) uniforms[i] = uni(draws);
        std::mt19937_64 rng(seed);
        const DensityUpdate up = densify_split(nx, err, static_cast<int>(budget), split_fraction, rng);
        if (static_cast<int64_t>(nx.size()) > cap) throw Error("bad-settings", "capacity");
        std::memcpy(nexels, nx.data(), nx.size() * sizeof(Nexel));
        std::memcpy(new_to_old, up.new_to_old.data(), up.new_to_old.size() * sizeof(int32_t));
        *n_out = static_cast<int64_t>(nx.size());
        *split_count = up.split_count;
    });
}

// nexel::prune (density.cpp:163-177); nexels compacted in place.
int ref_prune(double* nexels, int64_t n, double min_opacity, int32_t* new_to_old, int64_t* n_out) {
    return guarded([&] {
        std::vector<Nexel> nx(static_cast<size_t>(n));
        if (n) std::memcpy(nx.data(), nexels, n * sizeof(Nexel));
        const DensityUpdate up = prune(nx, min_opacity);
        if (!nx.empty()) std::memcpy(nexels, nx.data(), nx.size() * sizeof(Nexel));
        if (!up.new_to_old.empty()) std::memcpy(new_to_old, up.new_to_old.data(), up.new_to_old.size() * sizeof(int32_t));
        *n_out = static_cast<int64_t>(nx.size());
    });
}

// nexel::adam_remap_rows (adam.cpp:24-42): m / v of `rows_old` rows of `width` become
// `rows_new` rows (capacity) following new_to_old.
int ref_adam_remap_rows(double* m, double* v, int64_t rows_old, int64_t rows_new, const int32_t* new_to_old,
                        int64_t width) {
    return guarded([&] {
        AdamState st;
        st.m.assign(m, m + rows_old * width);
        st.v.assign(v, v + rows_old * width);
        std::vector<int32_t> map(new_to_old, new_to_old + rows_new);
        adam_remap_rows(st, map, static_cast<size_t>(width));
        std::memcpy(m, st.m.data(), st.m.size() * sizeof(double));
        std::memcpy(v, st.v.data(), st.v.size() * sizeof(double));
    });
}

}  // extern "C"
