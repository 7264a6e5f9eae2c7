// Synthetic render inputs shared by the CUDA path, the oracle and the bench
// (the `stump_like` scene and the ring cameras).
//
// Everything is generated on the host with libstdc++'s mt19937_64 /
// uniform_real_distribution / normal_distribution so that every consumer sees
// bit-identical inputs. Every stored primitive / field parameter is rounded
// through fp32 so the device's fp32 copies (SH, hash table, MLP) are exact.
//
// Field initialisation mirrors TextureField::init (texture_field.cpp:8-14 in
// the reference, via texture_field.hpp:22) and TextureMlp::init (mlp.cpp:13-22):
// uniform(-g, g) over the table in [level][row][feature] order, then one fresh
// normal_distribution per weight matrix with stddev sqrt(2 / fan_in).
// HashGridConfig::for_extent (hash_grid.cpp:15-24): base 1/extent, growth
// 32768^(1/(levels-1)).
#include "../../include/nexel_b200.h"

#include <cmath>
#include <cstring>
#include <random>

namespace {

struct V3 {
    double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross3(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm3(V3 a) { return std::sqrt(dot3(a, a)); }
inline V3 normalized3(V3 a) {
    const double n = norm3(a);
    return {a.x / n, a.y / n, a.z / n};
}
inline double f32(double x) { return static_cast<double>(static_cast<float>(x)); }

struct Gen {
    std::mt19937_64 g;
    std::uniform_real_distribution<double> u01{0.0, 1.0};
    double U() { return u01(g); }
};

void emit(Gen& G, double* out, V3 mu, V3 n, double sigma) {
    const double spin = 2.0 * M_PI * G.U();
    V3 j;
    j.x = G.U() - 0.5;
    j.y = G.U() - 0.5;
    j.z = G.U() - 0.5;
    const V3 m = normalized3(add(n, scale(0.1, j)));
    const V3 zhat{0.0, 0.0, 1.0};
    const V3 a = cross3(zhat, m);
    const double cz = dot3(zhat, m);
    const double an = norm3(a);
    double w1, x1, y1, z1;
    if (an < 1e-12) {
        w1 = 1.0;
        x1 = y1 = z1 = 0.0;
    } else {
        const double sh = std::sqrt((1.0 - cz) / 2.0);
        w1 = std::sqrt((1.0 + cz) / 2.0);
        x1 = a.x / an * sh;
        y1 = a.y / an * sh;
        z1 = a.z / an * sh;
    }
    const double w2 = std::cos(spin / 2.0), x2 = 0.0, y2 = 0.0, z2 = std::sin(spin / 2.0);
    // Hamilton product q1 (x) q2, (w, x, y, z).
    const double qw = w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2;
    const double qx = w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2;
    const double qy = w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2;
    const double qz = w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2;

    const double ls = std::log(sigma);
    const double lsx = ls + 0.6 * (G.U() - 0.5);
    const double lsy = ls + 0.6 * (G.U() - 0.5);
    const double p = 0.3 + 0.69 * G.U();
    const double op = std::log(p / (1.0 - p));  // inverse_sigmoid, vec_math.hpp:78
    const double gx = std::log(std::expm1(3.0 * G.U() + 1e-3));
    const double gy = std::log(std::expm1(3.0 * G.U() + 1e-3));

    out[0] = f32(mu.x);
    out[1] = f32(mu.y);
    out[2] = f32(mu.z);
    out[3] = f32(qw);
    out[4] = f32(qx);
    out[5] = f32(qy);
    out[6] = f32(qz);
    out[7] = f32(lsx);
    out[8] = f32(lsy);
    out[9] = f32(op);
    out[10] = f32(gx);
    out[11] = f32(gy);
    for (int k = 0; k < NX_SH_VALUES; ++k) {
        const double v = k < 3 ? 1.2 * (G.U() - 0.5) : 0.1 * (G.U() - 0.5);
        out[12 + k] = f32(v);
    }
}

}  // namespace

extern "C" void nx_settings_default(nx_settings* s) {
    std::memset(s, 0, sizeof(*s));
    s->top_k = 2;
    s->tile = 16;
    s->near_eps = 1e-3;
    s->alpha_max = 0.999;
    s->min_transmittance = 1e-4;
}

extern "C" int nx_synth_stump_like(int64_t n, double coverage, uint64_t seed, double ground_radius,
                                   int32_t log2_table, double grid_init, uint64_t field_seed,
                                   double* nexels, nx_settings* settings, nx_field_desc* field,
                                   double* table, double* w1, double* w2, double* w3) {
    if (n < 3 || coverage <= 0 || ground_radius <= 0 || log2_table < 1 || log2_table > 24)
        return NX_INVALID_ARGUMENT;
    const double Rg = ground_radius, Ro = 0.5, Ho = 0.8, Rd = 8.0, c = coverage;
    const int levels = 16, features = 2, hidden = 64;
    if (field) {
        field->levels = levels;
        field->log2_table = log2_table;
        field->features = features;
        field->n_hidden = hidden;
        field->base_scale = 1.0 / (2.0 * Rd);
        field->growth = std::pow(32768.0, 1.0 / (levels - 1));
    }
    if (settings) {
        nx_settings_default(settings);
        settings->top_k = 2;
        settings->background[0] = 0.1;
        settings->background[1] = 0.1;
        settings->background[2] = 0.12;
    }
    if (nexels) {
        Gen G{std::mt19937_64(seed)};
        const int64_t nG = static_cast<int64_t>(0.55 * static_cast<double>(n));
        const int64_t nO = static_cast<int64_t>(0.15 * static_cast<double>(n));
        const int64_t nD = n - nG - nO;
        const double sG = c * std::sqrt(M_PI * Rg * Rg / static_cast<double>(nG));
        const double sO = c * std::sqrt(2.0 * M_PI * Ro * Ho / static_cast<double>(nO));
        const double sD = c * std::sqrt(2.0 * M_PI * Rd * Rd / static_cast<double>(nD));
        double* out = nexels;
        for (int64_t i = 0; i < nG; ++i, out += NX_PARAMS_PER_NEXEL) {
            const double r = Rg * std::sqrt(G.U());
            const double th = 2.0 * M_PI * G.U();
            emit(G, out, {r * std::cos(th), r * std::sin(th), 0.0}, {0.0, 0.0, 1.0}, sG);
        }
        for (int64_t i = 0; i < nO; ++i, out += NX_PARAMS_PER_NEXEL) {
            const double th = 2.0 * M_PI * G.U();
            const double z = Ho * G.U();
            emit(G, out, {Ro * std::cos(th), Ro * std::sin(th), z}, {std::cos(th), std::sin(th), 0.0},
                 sO);
        }
        for (int64_t i = 0; i < nD; ++i, out += NX_PARAMS_PER_NEXEL) {
            const double z = G.U();
            const double th = 2.0 * M_PI * G.U();
            const double r = std::sqrt(1.0 - z * z);
            const V3 p{Rd * (r * std::cos(th)), Rd * (r * std::sin(th)), Rd * z};
            const double pn = norm3(p);
            emit(G, out, p, {-p.x / pn, -p.y / pn, -p.z / pn}, sD);
        }
    }
    if (table || w1 || w2 || w3) {
        if (!(table && w1 && w2 && w3)) return NX_INVALID_ARGUMENT;
        std::mt19937_64 rng(field_seed);
        const size_t n_table = static_cast<size_t>(levels) * (size_t(1) << log2_table) * features;
        std::uniform_real_distribution<double> dist(-grid_init, grid_init);
        for (size_t i = 0; i < n_table; ++i) table[i] = f32(dist(rng));
        const int n_in = levels * features;
        auto fill = [&rng](double* w, size_t count, int fan_in) {
            std::normal_distribution<double> nd(0.0, std::sqrt(2.0 / fan_in));
            for (size_t i = 0; i < count; ++i) w[i] = f32(nd(rng));
        };
        fill(w1, static_cast<size_t>(hidden) * n_in, n_in);
        fill(w2, static_cast<size_t>(hidden) * hidden, hidden);
        fill(w3, static_cast<size_t>(NX_SH_VALUES) * hidden, hidden);
    }
    return NX_OK;
}

// Ring camera i of n (OpenCV look-at as synthetic.cpp:44-65).
extern "C" int nx_synth_ring_camera(int index, int n_views, int width, int height, nx_camera* out) {
    if (n_views < 1 || width < 1 || height < 1 || !out) return NX_INVALID_ARGUMENT;
    const double th = 2.0 * M_PI * index / n_views + 0.37;
    const V3 eye{3.0 * std::cos(th), 3.0 * std::sin(th), 1.2 + 0.2 * std::sin(3.0 * th)};
    const V3 target{0.0, 0.0, 0.4};
    const V3 fwd = normalized3(sub(target, eye));
    const V3 right = normalized3(cross3(fwd, V3{0.0, 0.0, 1.0}));
    const V3 down = cross3(fwd, right);
    std::memset(out, 0, sizeof(*out));
    out->width = width;
    out->height = height;
    out->fx = out->fy = 0.8 * width;
    out->cx = width / 2.0;
    out->cy = height / 2.0;
    const V3 rows[3] = {right, down, fwd};
    for (int r = 0; r < 3; ++r) {
        out->R[r * 3 + 0] = rows[r].x;
        out->R[r * 3 + 1] = rows[r].y;
        out->R[r * 3 + 2] = rows[r].z;
        out->t[r] = -dot3(rows[r], eye);
    }
    return NX_OK;
}
