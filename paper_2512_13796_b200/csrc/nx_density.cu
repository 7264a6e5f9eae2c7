// Density control on the device scene (density.cpp:102-177) and the optimizer-row
// remap that follows it (adam_remap_rows, adam.cpp:24-42; trainer.cpp:324-332):
// elementwise kernels for the keys / flags / children, the library's stable radix sort
// and scan for the selection and the compaction, and gathers into the new layouts
// (the fp64 geometry is SoA with the nexel count as its stride, so every row moves).
#include <cmath>

#include "nx_internal.cuh"

namespace nx {

namespace {

constexpr int kT = 256;

__global__ void prune_flags_kernel(const double* geom, int64_t n, double min_opacity, int32_t* flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = sigmoid(geom[9 * n + i]) < min_opacity ? 0 : 1;  // density.cpp:168
}

// rows of the new layout from new_to_old (-1: left for the caller / zero)
__global__ void gather_geom_kernel(const double* geom, int64_t n, double* out, int64_t n_new, const int32_t* n2o) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_new) return;
    const int32_t src = n2o[i];
    for (int k = 0; k < kGeomFields; ++k) out[k * n_new + i] = src >= 0 ? geom[k * n + src] : 0.0;
}

__global__ void gather_rows_f32_kernel(const float* in, float* out, int64_t n_new, int width, const int32_t* n2o) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n_new * width) return;
    const int64_t i = e / width;
    const int32_t src = n2o[i];
    out[e] = src >= 0 ? in[static_cast<int64_t>(src) * width + (e - i * width)] : 0.f;
}

// adam_remap_rows: new rows take the source row's moments, fresh rows zero
__global__ void gather_rows_f64_kernel(const double* in, double* out, int64_t n_new, int width, const int32_t* n2o) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n_new * width) return;
    const int64_t i = e / width;
    const int32_t src = n2o[i];
    out[e] = src >= 0 ? in[static_cast<int64_t>(src) * width + (e - i * width)] : 0.0;
}

__global__ void compact_map_kernel(const int32_t* flags, const int32_t* pos, int64_t n, int32_t* n2o) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && flags[i]) n2o[pos[i]] = static_cast<int32_t>(i);
}

// sampling keys u^(1/e) (density.cpp:117-124) as ascending 64-bit sort keys (largest
// key first); non-positive errors sort last
__global__ void split_keys_kernel(const double* errors, const double* uniforms, int64_t n, uint64_t* keys,
                                  uint32_t* ids, unsigned long long* n_keys) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double e = errors[i];
    uint64_t key = ~0ull;
    if (e > 0.0) {
        key = ~depth_key(pow(uniforms[i], 1.0 / e));
        atomicAdd(n_keys, 1ull);
    }
    keys[i] = key;
    ids[i] = static_cast<uint32_t>(i);
}

// children of the selected parents (density.cpp:137-156): geometry in the old layout's
// rows (the parent slot) and the appended slot n + rank
__global__ void split_children_kernel(double* geom_new, int64_t n_new, const double* geom_old, int64_t n,
                                      const int32_t* parents, int64_t count) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    const int64_t j = parents[r];
    const double* g = geom_old;
    const double qw = g[3 * n + j], qx = g[4 * n + j], qy = g[5 * n + j], qz = g[6 * n + j];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz), inv = 1.0 / qn;  // activate (primitive.cpp:65-67)
    const double w = inv * qw, x = inv * qx, y = inv * qy, z = inv * qz;
    const double c0[3] = {1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)};  // R.col(0)
    const double c1[3] = {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)};  // R.col(1)
    const double sx = exp(g[7 * n + j]), sy = exp(g[8 * n + j]);
    double off[3];
    double ls[2] = {g[7 * n + j], g[8 * n + j]};
    if (sx >= sy) {
        for (int k = 0; k < 3; ++k) off[k] = (sx / 2.0) * c0[k];
        ls[0] = log(sx / 2.0);
    } else {
        for (int k = 0; k < 3; ++k) off[k] = (sy / 2.0) * c1[k];
        ls[1] = log(sy / 2.0);
    }
    const int64_t a = j, b = n + r;  // child, other
    for (int k = 0; k < kGeomFields; ++k) {
        const double v = g[k * n + j];
        geom_new[k * n_new + a] = v;
        geom_new[k * n_new + b] = v;
    }
    for (int k = 0; k < 2; ++k) {
        geom_new[(7 + k) * n_new + a] = ls[k];
        geom_new[(7 + k) * n_new + b] = ls[k];
    }
    for (int k = 0; k < 3; ++k) {
        geom_new[k * n_new + a] = g[k * n + j] + off[k];
        geom_new[k * n_new + b] = g[k * n + j] - off[k];
    }
}

__global__ void copy_sh_rows_kernel(float* sh, const int32_t* parents, int64_t n, int64_t count) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= count * NX_SH_VALUES) return;
    const int64_t r = e / NX_SH_VALUES;
    const int k = static_cast<int>(e - r * NX_SH_VALUES);
    sh[(n + r) * NX_SH_VALUES + k] = sh[static_cast<int64_t>(parents[r]) * NX_SH_VALUES + k];
}

__global__ void split_map_kernel(int32_t* n2o, int64_t n, const int32_t* parents, int64_t count) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) n2o[i] = static_cast<int32_t>(i);
    if (i < count) n2o[n + i] = -1;
}

__global__ void split_map_parents_kernel(int32_t* n2o, const int32_t* parents, int64_t count) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < count) n2o[parents[r]] = -1;
}

unsigned nb(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, (n + kT - 1) / kT)); }

}  // namespace

void launch_prune_flags(const double* geom, int64_t n, double min_opacity, int32_t* flags, cudaStream_t s) {
    count_launch();
    prune_flags_kernel<<<nb(n), kT, 0, s>>>(geom, n, min_opacity, flags);
}
void launch_compact_map(const int32_t* flags, const int32_t* pos, int64_t n, int32_t* n2o, cudaStream_t s) {
    count_launch();
    compact_map_kernel<<<nb(n), kT, 0, s>>>(flags, pos, n, n2o);
}
void launch_gather_geom(const double* geom, int64_t n, double* out, int64_t n_new, const int32_t* n2o, cudaStream_t s) {
    count_launch();
    gather_geom_kernel<<<nb(n_new), kT, 0, s>>>(geom, n, out, n_new, n2o);
}
void launch_gather_rows_f32(const float* in, float* out, int64_t n_new, int width, const int32_t* n2o, cudaStream_t s) {
    count_launch();
    gather_rows_f32_kernel<<<nb(n_new * width), kT, 0, s>>>(in, out, n_new, width, n2o);
}
void launch_gather_rows_f64(const double* in, double* out, int64_t n_new, int width, const int32_t* n2o,
                            cudaStream_t s) {
    count_launch();
    gather_rows_f64_kernel<<<nb(n_new * width), kT, 0, s>>>(in, out, n_new, width, n2o);
}
void launch_split_keys(const double* errors, const double* uniforms, int64_t n, uint64_t* keys, uint32_t* ids,
                       unsigned long long* n_keys, cudaStream_t s) {
    count_launch();
    split_keys_kernel<<<nb(n), kT, 0, s>>>(errors, uniforms, n, keys, ids, n_keys);
}
void launch_split_children(double* geom_new, int64_t n_new, const double* geom_old, int64_t n, float* sh,
                           const int32_t* parents, int64_t count, int32_t* n2o, cudaStream_t s) {
    count_launch(5);
    split_map_kernel<<<nb(std::max(n, count)), kT, 0, s>>>(n2o, n, parents, count);
    split_map_parents_kernel<<<nb(count), kT, 0, s>>>(n2o, parents, count);
    gather_geom_kernel<<<nb(n_new), kT, 0, s>>>(geom_old, n, geom_new, n_new, n2o);  // untouched rows
    split_children_kernel<<<nb(count), kT, 0, s>>>(geom_new, n_new, geom_old, n, parents, count);
    copy_sh_rows_kernel<<<nb(count * NX_SH_VALUES), kT, 0, s>>>(sh, parents, n, count);
}

}  // namespace nx
