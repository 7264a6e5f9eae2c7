// GPU drop-in of nexel::render_backward (paper_2512_13796_b200/host/renderer_b200.cpp)
// against the reference's own render_backward (renderer.cpp:251-401, compiled in the
// same library under the name nexel_ref_render_backward) on the same forward output:
// random scenes from the reference's test helpers (tests/helpers.hpp:88-125),
// K = 0..4, with and without the blended-error bookkeeping; and the drop-in render after
// the Scene is edited in place (same arrays: the pass that starts on the cached device
// scene must be redone from the new content) against the reference's own render.
// Built by `make dropin`.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "helpers.hpp"
#include "nexel/renderer.hpp"

namespace nexel {
RenderResult nexel_ref_render(const Scene& scene, const Camera& cam);
void nexel_ref_render_backward(const Scene& scene, const Camera& cam, const FrameBuffers& fb,
                               const UpstreamGrads& up, SceneGrads& grads, const double* err_pixel,
                               std::vector<double>* blended_error);
}

using namespace nexel;
using namespace testutil;

namespace {

// max |a - b| / max |b| over one gradient array
double normwise(const std::vector<double>& a, const std::vector<double>& b) {
    double err = 0, scale = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        err = std::max(err, std::abs(a[i] - b[i]));
        scale = std::max(scale, std::abs(b[i]));
    }
    return scale > 0 ? err / scale : err;
}

std::vector<double> flat(const std::vector<PrimitiveGrad>& p) {
    std::vector<double> out(p.size() * 60);
    for (size_t i = 0; i < p.size(); ++i) std::memcpy(&out[i * 60], &p[i], 60 * sizeof(double));
    return out;
}

}  // namespace

TEST_CASE("drop-in render_backward equals the reference's on the forward output") {
    for (int k : {0, 1, 2, 4}) {
        std::mt19937_64 g(700 + k);
        const Scene scene = random_scene(g, 50, k);
        const Camera cam = orbit_camera(g, 40, 50.0, 3.0);
        const RenderResult rr = render(scene, cam);  // the drop-in forward (GPU)
        const size_t npix = static_cast<size_t>(cam.width) * cam.height;
        std::vector<double> df(npix * 3), dw(npix * k), dt(npix * k * 3), err(npix);
        for (double& v : df) v = urand(g, -1, 1);
        for (double& v : dw) v = urand(g, -1, 1);
        for (double& v : dt) v = urand(g, -1, 1);
        for (double& v : err) v = urand(g, 0, 1);
        UpstreamGrads up;
        up.d_final = df.data();
        up.d_weights = k ? dw.data() : nullptr;
        up.d_texture = k ? dt.data() : nullptr;

        SceneGrads ours, ref;
        ours.allocate(scene);
        ref.allocate(scene);
        std::vector<double> be_ours(scene.nexels.size(), 0.0), be_ref(scene.nexels.size(), 0.0);
        render_backward(scene, cam, rr.fb, up, ours, err.data(), &be_ours);
        nexel_ref_render_backward(scene, cam, rr.fb, up, ref, err.data(), &be_ref);

        INFO("k = " << k);
        CHECK(normwise(flat(ours.prims), flat(ref.prims)) <= 1e-5);
        CHECK(normwise(ours.field.table, ref.field.table) <= 1e-5);
        CHECK(normwise(ours.field.w1, ref.field.w1) <= 1e-5);
        CHECK(normwise(ours.field.w2, ref.field.w2) <= 1e-5);
        CHECK(normwise(ours.field.w3, ref.field.w3) <= 1e-5);
        CHECK(normwise(be_ours, be_ref) <= 1e-6);
        double mx = 0;
        for (double v : flat(ref.prims)) mx = std::max(mx, std::abs(v));
        CHECK(mx > 0);
    }
}

TEST_CASE("drop-in render_backward accumulates and reports unallocated gradients") {
    std::mt19937_64 g(811);
    const Scene scene = random_scene(g, 20, 2);
    const Camera cam = orbit_camera(g, 24, 30.0, 3.0);
    const RenderResult rr = render(scene, cam);
    std::vector<double> df(static_cast<size_t>(cam.width) * cam.height * 3, 0.5);
    UpstreamGrads up;
    up.d_final = df.data();
    SceneGrads once, twice;
    once.allocate(scene);
    twice.allocate(scene);
    render_backward(scene, cam, rr.fb, up, once);
    render_backward(scene, cam, rr.fb, up, twice);
    render_backward(scene, cam, rr.fb, up, twice);
    std::vector<double> a = flat(once.prims), b = flat(twice.prims);
    for (double& v : a) v *= 2;
    CHECK(normwise(b, a) <= 1e-6);
    SceneGrads empty;
    CHECK_THROWS_AS(render_backward(scene, cam, rr.fb, up, empty), Error);
}

namespace {

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

void check_same_frame(const RenderResult& ours, const RenderResult& ref) {
    CHECK(ours.fb.ids == ref.fb.ids);
    CHECK(max_abs_diff(ours.fb.depths, ref.fb.depths) <= 1e-9);
    CHECK(max_abs_diff(ours.fb.weights, ref.fb.weights) <= 1e-9);
    CHECK(max_abs_diff(ours.fb.final_img, ref.fb.final_img) <= 1e-6);
    CHECK(max_abs_diff(ours.fb.texture, ref.fb.texture) <= 1e-6);
}

}  // namespace

TEST_CASE("drop-in render follows in-place edits of the Scene") {
    std::mt19937_64 g(913);
    Scene scene = random_scene(g, 80, 2);
    const Camera cam = orbit_camera(g, 48, 50.0, 3.0);
    const RenderResult first = render(scene, cam);  // binds the device scene
    check_same_frame(first, nexel_ref_render(scene, cam));
    const void* nexels_before = scene.nexels.data();
    // geometry, opacity and colour of some primitives, and the hash table, edited in place
    for (size_t i = 0; i < scene.nexels.size(); i += 3) {
        scene.nexels[i].opacity_raw += 1.5;
        scene.nexels[i].mu.x += 0.05;
        scene.nexels[i].sh[0] -= 0.3;
    }
    for (size_t i = 0; i < scene.field.grid.table.size(); i += 7) scene.field.grid.table[i] += 0.05;
    REQUIRE(scene.nexels.data() == nexels_before);
    const RenderResult second = render(scene, cam);
    const RenderResult ref = nexel_ref_render(scene, cam);
    check_same_frame(second, ref);
    CHECK(max_abs_diff(second.fb.final_img, first.fb.final_img) > 1e-3);  // the edit shows
    // the same content again, unchanged arrays: the speculative pass stands
    const RenderResult third = render(scene, cam);
    CHECK(third.fb.ids == second.fb.ids);
    CHECK(third.fb.final_img == second.fb.final_img);
    // a copy (other arrays, same content) renders the same frame
    const Scene copy = scene;
    const RenderResult fourth = render(copy, cam);
    CHECK(fourth.fb.ids == second.fb.ids);
    CHECK(fourth.fb.final_img == second.fb.final_img);
}
