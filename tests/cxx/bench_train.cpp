// Training-loop throughput of the GPU-backed nexel::train (host/trainer_b200.cpp) against
// the reference's own train (nexel_ref_train, CPU) on one synthetic bundle
// (three_quad_job at 256x256, 16 views, 4000 seed points; budget 20000 primitives with
// densification on). The GPU run trains `iters` iterations; the reference a bounded
// number (its per-iteration wall time, from the on_iteration hook, is the figure).
// Prints one JSON line. Usage: bench_train [iters] [ref_iters]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "nexel/synthetic.hpp"
#include "nexel/trainer.hpp"

namespace nexel {
TrainResult nexel_ref_train(const Bundle& bundle, const TrainConfig& cfg, const TrainHooks& hooks);
}

using namespace nexel;

int main(int argc, char** argv) {
    const int iters = argc > 1 ? std::atoi(argv[1]) : 300;
    const int ref_iters = argc > 2 ? std::atoi(argv[2]) : 6;
    const std::string dir = (std::filesystem::temp_directory_path() / "nexel_bench_train_bundle").string();
    SynthJob job = three_quad_job();
    job.n_views = 16;
    job.n_test = 2;
    job.resolution = 256;
    job.cloud_points = 4000;
    job.seed = 7;
    make_synthetic_bundle(job, dir);
    const Bundle bundle = load_bundle(dir);

    TrainConfig cfg;
    cfg.budget = 20000;
    cfg.seed = 3;
    cfg.top_k = 2;
    cfg.densify_start = 50;
    cfg.densify_every = 50;
    cfg.densify_end = 100000;
    cfg.grid_log2_table = 18;

    std::vector<double> gpu_walls;
    double gpu_wall = 0.0, ref_wall = 0.0;
    int gpu_count = 0, ref_count = 0, gpu_prims = 0;
    double gpu_loss = 0.0, ref_loss = 0.0;
    {
        cfg.iterations = iters;
        TrainHooks h;
        h.on_iteration = [&](int, const LossTerms& t, int n, double wall) {
            gpu_wall += wall;
            gpu_walls.push_back(wall);
            gpu_prims = n;
            gpu_loss = t.total;
        };
        const auto t0 = std::chrono::steady_clock::now();
        train(bundle, cfg, h);
        gpu_count = iters;
        const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "gpu: %d iterations in %.2f s (hooks %.2f s)\n", iters, total, gpu_wall);
    }
    {
        cfg.iterations = ref_iters;
        TrainHooks h;
        h.on_iteration = [&](int, const LossTerms& t, int, double wall) {
            ref_wall += wall;
            ref_loss = t.total;
            ++ref_count;
        };
        nexel_ref_train(bundle, cfg, h);
    }
    // like for like: the GPU's own first ref_iters iterations (same scene sizes as the
    // reference's), plus its whole-run rate
    double gpu_first = 0.0;
    for (int i = 0; i < ref_count && i < static_cast<int>(gpu_walls.size()); ++i) gpu_first += gpu_walls[i];
    const double gpu_it = gpu_count / gpu_wall, ref_it = ref_count / ref_wall, gpu_first_it = ref_count / gpu_first;
    std::printf(
        "{\"metric\": \"training iterations/s (nexel::train, synthetic three-quad bundle 256x256, 16 views, "
        "budget 20000, densify every 50)\", \"gpu_iters_per_s\": %.2f, \"gpu_iterations\": %d, \"gpu_final_prims\": %d, "
        "\"gpu_final_loss\": %.6g, \"gpu_first_iters_per_s\": %.2f, \"reference_iters_per_s\": %.4f, "
        "\"reference_iterations\": %d, \"reference_loss_at_end\": %.6g, \"speedup_same_iterations\": %.1f}\n",
        gpu_it, gpu_count, gpu_prims, gpu_loss, gpu_first_it, ref_it, ref_count, ref_loss, gpu_first_it / ref_it);
    std::filesystem::remove_all(dir);
    return 0;
}
