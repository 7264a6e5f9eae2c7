// Driver of the data-parallel nexel::train test (tests/test_gpu_dp_train.py): trains a
// small synthetic bundle (three_quad_job, 64x64) through the GPU-backed nexel::train —
// one process per rank, NEXEL_DP_* from the environment — and prints one line with the
// digest of the resulting scene (every fp64 parameter and the field), the primitive
// count and the last mean loss. Usage: dp_train <bundle_dir> <iterations> <single_view>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nexel/synthetic.hpp"
#include "nexel/trainer.hpp"

using namespace nexel;

namespace {
uint64_t fnv(uint64_t h, const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const std::string dir = argv[1];
    const int iters = std::atoi(argv[2]);
    const bool single_view = std::atoi(argv[3]) != 0;
    SynthJob job = three_quad_job();
    job.n_views = 8;
    job.n_test = 2;
    job.resolution = 64;
    job.cloud_points = 600;
    job.seed = 7;
    make_synthetic_bundle(job, dir);
    Bundle bundle = load_bundle(dir);
    if (single_view) bundle.train_views.resize(1);

    TrainConfig cfg;
    cfg.iterations = iters;
    cfg.budget = 3000;
    cfg.seed = 3;
    cfg.top_k = 2;
    cfg.densify_start = 4;
    cfg.densify_every = 4;
    cfg.densify_end = 1000;
    cfg.grid_log2_table = 14;
    const TrainResult r = train(bundle, cfg);
    uint64_t h = 1469598103934665603ull;
    h = fnv(h, r.scene.nexels.data(), r.scene.nexels.size() * sizeof(Nexel));
    h = fnv(h, r.scene.field.grid.table.data(), r.scene.field.grid.table.size() * sizeof(double));
    for (const auto* w : {&r.scene.field.mlp.w1, &r.scene.field.mlp.w2, &r.scene.field.mlp.w3})
        h = fnv(h, w->data(), w->size() * sizeof(double));
    for (const AdamState& a : r.optimizer) {
        h = fnv(h, a.m.data(), a.m.size() * sizeof(double));
        h = fnv(h, a.v.data(), a.v.size() * sizeof(double));
    }
    std::printf("digest %016llx nexels %zu loss %.17g\n", static_cast<unsigned long long>(h), r.scene.nexels.size(),
                r.last_loss.total);
    return 0;
}
