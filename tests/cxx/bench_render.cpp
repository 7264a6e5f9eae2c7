// Throughput of the reference API's render path through the C++ drop-in:
// nexel::render(scene, cam) (renderer.hpp:28, the call cmd_render and mean_psnr make,
// nexel_cli.cpp:113-121, trainer.cpp:215-229) with the Scene held in host doubles and the
// RenderResult returned in host doubles, at BASELINE config 2 (stump_like 400K nexels,
// 1920x1080, K = 2, ring view 0). Each timed call includes the scene fingerprint, the
// device passes, the downloads and the widening into the FrameBuffers vectors (whose
// allocation is part of the API: RenderResult is returned by value).
// Prints one JSON line. Usage: bench_render [frames] [n_nexels] [width] [height]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "nexel/renderer.hpp"
#include "../../include/nexel_b200.h"

using namespace nexel;

int main(int argc, char** argv) {
    const int frames = argc > 1 ? std::atoi(argv[1]) : 10;
    const int64_t n = argc > 2 ? std::atoll(argv[2]) : 400000;
    const int W = argc > 3 ? std::atoi(argv[3]) : 1920, H = argc > 4 ? std::atoi(argv[4]) : 1080;

    Scene scene;
    nx_settings st;
    nx_field_desc fd;
    if (nx_synth_stump_like(n, 1.0, 2512, 4.0, 20, 1e-4, 2513, nullptr, nullptr, &fd, nullptr, nullptr, nullptr,
                            nullptr) != NX_OK)
        return 2;
    scene.nexels.resize(static_cast<size_t>(n));
    HashGridConfig g;
    g.levels = fd.levels;
    g.log2_table = fd.log2_table;
    g.features = fd.features;
    g.base_scale = fd.base_scale;
    g.growth = fd.growth;
    scene.field.grid.cfg = g;
    scene.field.grid.allocate();
    scene.field.mlp.n_in = fd.levels * fd.features;
    scene.field.mlp.n_hidden = fd.n_hidden;
    scene.field.mlp.w1.resize(static_cast<size_t>(fd.n_hidden) * scene.field.mlp.n_in);
    scene.field.mlp.w2.resize(static_cast<size_t>(fd.n_hidden) * fd.n_hidden);
    scene.field.mlp.w3.resize(static_cast<size_t>(48) * fd.n_hidden);
    if (nx_synth_stump_like(n, 1.0, 2512, 4.0, 20, 1e-4, 2513, &scene.nexels[0].mu.x, &st, &fd,
                            scene.field.grid.table.data(), scene.field.mlp.w1.data(), scene.field.mlp.w2.data(),
                            scene.field.mlp.w3.data()) != NX_OK)
        return 2;
    scene.settings.top_k = st.top_k;
    scene.settings.background = {st.background[0], st.background[1], st.background[2]};
    scene.extent = 8.0;
    nx_camera nc;
    nx_synth_ring_camera(0, 256, W, H, &nc);
    Camera cam;
    cam.width = nc.width;
    cam.height = nc.height;
    cam.fx = nc.fx;
    cam.fy = nc.fy;
    cam.cx = nc.cx;
    cam.cy = nc.cy;
    for (int r = 0; r < 3; ++r) {
        for (int k = 0; k < 3; ++k) cam.R.m[r][k] = nc.R[r * 3 + k];
        cam.t[r] = nc.t[r];
    }

    double sum_final = 0.0;
    for (int w = 0; w < 2; ++w) {  // first call uploads the scene
        RenderResult r = render(scene, cam);
        sum_final = 0.0;
        for (double v : r.fb.final_img) sum_final += v;
    }
    std::vector<double> ms;
    for (int f = 0; f < frames; ++f) {
        const auto t0 = std::chrono::steady_clock::now();
        RenderResult r = render(scene, cam);
        const auto t1 = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    double tot = 0.0;
    for (double v : ms) tot += v;
    std::printf("{\"metric\": \"nexel::render frames/s (reference C++ API, host Scene + FrameBuffers)\", "
                "\"value\": %.3f, \"unit\": \"frames/s\", \"ms_per_frame\": %.3f, \"frames\": %d, "
                "\"n_nexels\": %lld, \"width\": %d, \"height\": %d, \"sum_final\": %.9f}\n",
                1000.0 * frames / tot, tot / frames, frames, static_cast<long long>(n), W, H, sum_final);
    return 0;
}
