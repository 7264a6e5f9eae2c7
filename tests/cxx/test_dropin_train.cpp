// The GPU-backed nexel::train (paper_2512_13796_b200/host/trainer_b200.cpp) against the
// reference's own train (trainer.cpp compiled in place, exported as nexel_ref_train) on
// the reference's synthetic bundles (three_quad_job, as test_train.cpp's tiny_bundle):
// the same view sequence and densify schedule, primitive counts equal at every
// iteration, loss terms and final parameters within the drift the fp32 render path
// allows, the same optimizer step counts; and bit-identical results run to run.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "helpers.hpp"

#include "nexel/checkpoint.hpp"
#include "nexel/synthetic.hpp"
#include "nexel/trainer.hpp"

#include <cmath>
#include <cstdio>

namespace nexel {
TrainResult nexel_ref_train(const Bundle& bundle, const TrainConfig& cfg, const TrainHooks& hooks);
}

using namespace nexel;
using namespace testutil;

namespace {

const Bundle& bundle_of(int resolution, int views, int cloud, uint64_t seed) {
    static TempDir tmp;
    static std::vector<std::pair<std::string, Bundle>> made;
    const std::string key = std::to_string(resolution) + "_" + std::to_string(views) + "_" + std::to_string(cloud);
    for (auto& m : made)
        if (m.first == key) return m.second;
    SynthJob job = three_quad_job();
    job.n_views = views;
    job.n_test = 1;
    job.resolution = resolution;
    job.cloud_points = cloud;
    job.seed = seed;
    const std::string dir = tmp.file("b" + key);
    make_synthetic_bundle(job, dir);
    made.emplace_back(key, load_bundle(dir));
    return made.back().second;
}

struct Trace {
    std::vector<LossTerms> terms;
    std::vector<int> counts;
};

TrainResult run(bool gpu, const Bundle& b, const TrainConfig& cfg, Trace* tr) {
    TrainHooks hooks;
    if (tr)
        hooks.on_iteration = [tr](int, const LossTerms& t, int n, double) {
            tr->terms.push_back(t);
            tr->counts.push_back(n);
        };
    return gpu ? train(b, cfg, hooks) : nexel_ref_train(b, cfg, hooks);
}

double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    double scale = 0.0, err = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        scale = std::max(scale, std::abs(b[i]));
        err = std::max(err, std::abs(a[i] - b[i]));
    }
    return scale > 0 ? err / scale : err;
}

TrainConfig config(int iterations, int budget) {
    TrainConfig cfg;
    cfg.iterations = iterations;
    cfg.budget = budget;
    cfg.seed = 4;
    cfg.top_k = 2;
    cfg.background = {0.08, 0.08, 0.1};
    cfg.densify_start = 2;
    cfg.densify_end = iterations - 2;
    cfg.densify_every = 2;
    cfg.split_fraction = 0.4;
    cfg.grid_levels = 4;
    cfg.grid_log2_table = 6;
    return cfg;
}

void compare(const Bundle& b, const TrainConfig& cfg, double loss_rtol, double param_rtol) {
    Trace tg, tr;
    const TrainResult g = run(true, b, cfg, &tg);
    const TrainResult r = run(false, b, cfg, &tr);
    REQUIRE(tg.counts.size() == tr.counts.size());
    CHECK(tg.counts == tr.counts);
    double worst = 0.0;
    for (size_t i = 0; i < tg.terms.size(); ++i) {
        const double rel = std::abs(tg.terms[i].total - tr.terms[i].total) / std::abs(tr.terms[i].total);
        worst = std::max(worst, rel);
        CHECK(std::abs(tg.terms[i].image - tr.terms[i].image) <= loss_rtol * std::abs(tr.terms[i].image));
    }
    CHECK(worst <= loss_rtol);
    REQUIRE(g.scene.nexels.size() == r.scene.nexels.size());
    const double prel = max_rel(pack_scene(g.scene), pack_scene(r.scene));
    CHECK(prel <= param_rtol);
    for (int k = 0; k < kGroupCount; ++k) {
        CHECK(g.optimizer[k].step == r.optimizer[k].step);
        CHECK(g.optimizer[k].m.size() == r.optimizer[k].m.size());
    }
    CHECK(g.extra.iteration == r.extra.iteration);
    std::printf("  %zu iterations, final count %d: worst loss rel diff %.2e, param rel diff %.2e\n",
                tg.terms.size(), tg.counts.empty() ? 0 : tg.counts.back(), worst, prel);
}

}  // namespace

TEST_CASE("GPU train follows the reference on the tiny bundle (densify + prune on)") {
    compare(bundle_of(24, 6, 80, 11), config(12, 24), 1e-5, 1e-4);
}

TEST_CASE("GPU train follows the reference on a larger bundle") {
    TrainConfig cfg = config(16, 200);
    cfg.grid_levels = 8;
    cfg.grid_log2_table = 10;
    compare(bundle_of(64, 8, 400, 3), cfg, 1e-5, 1e-4);
}

TEST_CASE("GPU train with the reference field shape (tensor-core field backward)") {
    TrainConfig cfg = config(8, 120);
    cfg.grid_levels = 16;
    cfg.grid_log2_table = 12;
    // the tensor-core field backward forms the MLP products from a 3-term bf16 split
    // (~1e-5 relative) and Adam's per-entry normalisation turns that into full-size step
    // differences on entries whose gradients are near zero: looser bounds here (the SIMT
    // field shapes above agree to ~1e-8)
    compare(bundle_of(48, 6, 200, 5), cfg, 1e-4, 1e-2);
}

TEST_CASE("GPU train is bit-reproducible and zero iterations return the initialisation") {
    const Bundle& b = bundle_of(24, 6, 80, 11);
    const TrainConfig cfg = config(10, 24);
    const TrainResult r1 = run(true, b, cfg, nullptr);
    const TrainResult r2 = run(true, b, cfg, nullptr);
    CHECK(pack_scene(r1.scene) == pack_scene(r2.scene));
    for (int k = 0; k < kGroupCount; ++k) {
        CHECK(r1.optimizer[k].m == r2.optimizer[k].m);
        CHECK(r1.optimizer[k].v == r2.optimizer[k].v);
    }
    TrainConfig zero = cfg;
    zero.iterations = 0;
    const TrainResult z = run(true, b, zero, nullptr);
    std::mt19937_64 rng(zero.seed);
    CHECK(pack_scene(z.scene) == pack_scene(initialize_scene(b, zero, rng)));
}
