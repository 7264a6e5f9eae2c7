// Adam on the device scene (adam_step, adam.cpp:9-22) for the trainer's parameter
// groups (trainer.cpp:238-323): position, quat, log-scale, opacity, gamma (the fp64
// geometry rows), SH DC / rest (fp32 n x 48), hash table, w1, w2, w3 (fp32). Moments
// are fp64 like the reference's AdamState; each group is one elementwise kernel over
// its parameters, reading the fp64 SceneGrads in place (PrimitiveGrad n x 60). The
// groups the scene stores in fp32 are stepped on fp64 master copies (the optimizer's),
// whose rounding refreshes the scene's fp32 values — so the trajectory follows the
// reference's fp64 parameters instead of re-rounding them every step.
#include <cmath>

#include "nx_internal.cuh"

namespace nx {

namespace {

struct AdamArgs {
    double lr, beta1, beta2, eps, bc1, bc2;
};

__device__ __forceinline__ double adam_update(double p, double g, double& m, double& v, const AdamArgs& c) {
    m = c.beta1 * m + (1.0 - c.beta1) * g;
    v = c.beta2 * v + (1.0 - c.beta2) * g * g;
    const double m_hat = m / c.bc1;
    const double v_hat = v / c.bc2;
    return p - c.lr * m_hat / (sqrt(v_hat) + c.eps);
}

// geometry group: `width` fp64 rows starting at `row0` of the SoA geometry; PrimitiveGrad
// column col0 + k holds the gradient of row row0 + k.
__global__ void adam_geom_kernel(double* geom, int64_t n, int row0, int width, int col0, const double* g,
                                 double* m, double* v, AdamArgs c) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * width) return;
    const int64_t prim = i / width;
    const int k = static_cast<int>(i - prim * width);
    double* p = geom + static_cast<int64_t>(row0 + k) * n + prim;
    *p = adam_update(*p, g[prim * NX_PARAMS_PER_NEXEL + col0 + k], m[i], v[i], c);
}

// SH group: columns [c0, c0 + width) of the fp32 n x 48 array; master (n x width) holds
// the fp64 values
__global__ void adam_sh_kernel(float* sh, double* master, int64_t n, int c0, int width, const double* g, double* m,
                               double* v, AdamArgs c) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * width) return;
    const int64_t prim = i / width;
    const int k = static_cast<int>(i - prim * width);
    float* p = sh + prim * NX_SH_VALUES + c0 + k;
    const double x = adam_update(master ? master[i] : static_cast<double>(*p),
                                 g[prim * NX_PARAMS_PER_NEXEL + 12 + c0 + k], m[i], v[i], c);
    if (master) master[i] = x;
    *p = static_cast<float>(x);
}

// flat fp32 block (table, w1, w2, w3) + its fp64 master
__global__ void adam_flat_kernel(float* p, double* master, int64_t count, const double* g, double* m, double* v,
                                 AdamArgs c) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = adam_update(master ? master[i] : static_cast<double>(p[i]), g[i], m[i], v[i], c);
        if (master) master[i] = x;
        p[i] = static_cast<float>(x);
    }
}

// group values <-> the group's row layout: geometry rows of the SoA (fp64), SH columns
// or flat blocks (fp32 scene copy). to_rows: scene -> rows (widening), else rows -> scene
// (rounding to the scene's storage).
__global__ void group_io_kernel(int group, int64_t n, int64_t count, double* geom, float* sh, float* flat,
                                double* rows, int to_rows) {
    const int row0[5] = {0, 3, 7, 9, 10}, width[7] = {3, 4, 2, 1, 2, 3, 45};
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (group <= 4) {
            const int64_t prim = i / width[group];
            const int k = static_cast<int>(i - prim * width[group]);
            double* p = geom + static_cast<int64_t>(row0[group] + k) * n + prim;
            if (to_rows) rows[i] = *p;
            else *p = rows[i];
        } else if (group <= 6) {
            const int64_t prim = i / width[group];
            const int k = static_cast<int>(i - prim * width[group]);
            float* p = sh + prim * NX_SH_VALUES + (group == 5 ? 0 : 3) + k;
            if (to_rows) rows[i] = *p;
            else *p = static_cast<float>(rows[i]);
        } else {
            if (to_rows) rows[i] = flat[i];
            else flat[i] = static_cast<float>(rows[i]);
        }
    }
}

unsigned blocks_for(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32))); }

}  // namespace

// Group sizes in parameters (the AdamState sizes of trainer.cpp:238-250).
void adam_group_sizes(const SceneDev& sc, int64_t* sizes) {
    const int64_t n = sc.n;
    const int64_t nin = static_cast<int64_t>(sc.field.levels) * sc.field.features, nh = sc.field.n_hidden;
    const int64_t w[7] = {3, 4, 2, 1, 2, 3, 45};
    for (int gi = 0; gi < 7; ++gi) sizes[gi] = n * w[gi];
    sizes[7] = static_cast<int64_t>(sc.field.levels) * (int64_t(1) << sc.field.log2_table) * sc.field.features;
    sizes[8] = nh * nin;
    sizes[9] = nh * nh;
    sizes[10] = NX_SH_VALUES * nh;
}

void launch_group_io(int group, const SceneDev& sc, double* geom, float* sh, float* table, float* w1, float* w2,
                     float* w3, double* rows, bool to_rows, cudaStream_t s) {
    int64_t sizes[NX_NUM_GROUPS];
    adam_group_sizes(sc, sizes);
    if (sizes[group] == 0) return;
    float* flat = group == 7 ? table : group == 8 ? w1 : group == 9 ? w2 : w3;
    count_launch();
    group_io_kernel<<<blocks_for(sizes[group]), 256, 0, s>>>(group, sc.n, sizes[group], geom, sh, flat, rows,
                                                               to_rows ? 1 : 0);
}

void launch_adam_group(int group, const SceneDev& sc, double* geom, float* sh, float* table, float* w1, float* w2,
                       float* w3, const nx_grads& g, double* m, double* v, double* master, const nx_adam_config& cfg,
                       int64_t step, cudaStream_t s) {
    AdamArgs c;
    c.lr = cfg.lr;
    c.beta1 = cfg.beta1;
    c.beta2 = cfg.beta2;
    c.eps = cfg.eps;
    c.bc1 = 1.0 - std::pow(cfg.beta1, static_cast<double>(step));  // adam.cpp:13-14
    c.bc2 = 1.0 - std::pow(cfg.beta2, static_cast<double>(step));
    const int64_t n = sc.n;
    static const int row0[5] = {0, 3, 7, 9, 10}, width[5] = {3, 4, 2, 1, 2};
    count_launch();
    if (group <= 4) {
        const int64_t cnt = n * width[group];
        adam_geom_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(geom, n, row0[group], width[group],
                                                                                  row0[group], g.prims, m, v, c);
    } else if (group <= 6) {
        const int c0 = group == 5 ? 0 : 3, wd = group == 5 ? 3 : 45;
        const int64_t cnt = n * wd;
        adam_sh_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, s>>>(sh, master, n, c0, wd, g.prims, m, v,
                                                                                c);
    } else {
        int64_t sizes[NX_NUM_GROUPS];
        adam_group_sizes(sc, sizes);
        float* p = group == 7 ? table : group == 8 ? w1 : group == 9 ? w2 : w3;
        const double* gg = group == 7 ? g.table : group == 8 ? g.w1 : group == 9 ? g.w2 : g.w3;
        adam_flat_kernel<<<blocks_for(sizes[group]), 256, 0, s>>>(p, master, sizes[group], gg, m, v, c);
    }
}

}  // namespace nx
