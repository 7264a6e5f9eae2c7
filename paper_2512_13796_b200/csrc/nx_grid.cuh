// Hash-grid lookup helpers (grid_lookup, hash_grid.cpp:26-83; hash_cell,
// hash_grid.hpp:12-23) shared by the texture forward and the field backward:
// lattice position, floor and hashing in fp64/int64 (or 32-bit when the lattice
// coordinates fit), so that the same table rows as the reference are read.
#pragma once

#include "nx_internal.cuh"

namespace nx {
namespace {

constexpr int kLevels = 16;

struct TcConst {
    double level_scale[kLevels];  // HashGridConfig::level_scale by iterated product (hash_grid.cpp:7-13)
    float inv_level_scale[kLevels];
    double inv_level_scale2[kLevels];  // 1 / level_scale^2 (the fade's t-gradient)
};

__device__ __forceinline__ uint32_t map_positive32(long long x) {  // hash_grid.hpp:12-14
    return x > 0 ? static_cast<uint32_t>(2 * x - 1) : static_cast<uint32_t>(-2 * x);
}

// One level of grid_lookup (hash_grid.cpp:32-82): lattice cell in fp64/int64 like the
// reference, the 8 hashed corner rows (hash_cell, hash_grid.hpp:17-23) gathered, the
// fractional position and the level fade (downweight, hash_grid.hpp:28-31).
struct LevelFetch {
    float2 v[8];
    float fr0, fr1, fr2, dw;
};

// map_positive for |x| < 2^30: the 32-bit wrap of the reference's 64-bit value.
__device__ __forceinline__ uint32_t map_positive_small(int x) {
    return x > 0 ? (static_cast<uint32_t>(x) << 1) - 1u : static_cast<uint32_t>(-x) << 1;
}

// kSmall: every lattice coordinate of the query fits in 30 bits (checked per query),
// so the cell index and hash run in 32-bit integers with identical results.
template <bool kSmall>
__device__ __forceinline__ LevelFetch fetch_level(int l, double x0, double x1, double x2, const TcConst& cst,
                                                  const float2* __restrict__ tab, uint32_t T, uint32_t mask, float ft,
                                                  int no_downweight) {
    LevelFetch f;
    const double s = cst.level_scale[l];
    const double p0 = s * x0, p1 = s * x1, p2 = s * x2;
    const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
    f.fr0 = static_cast<float>(p0 - fl0);
    f.fr1 = static_cast<float>(p1 - fl1);
    f.fr2 = static_cast<float>(p2 - fl2);
    f.dw = 1.0f;
    if (!no_downweight) {
        const float r = ft * cst.inv_level_scale[l];
        f.dw = 1.0f - __expf(-r * r * 0.15915494309189535f);
    }
    uint32_t ax0, ax1, by0, by1, cz0, cz1;
    if (kSmall) {
        const int b0 = static_cast<int>(fl0), b1 = static_cast<int>(fl1), b2 = static_cast<int>(fl2);
        ax0 = map_positive_small(b0);
        ax1 = map_positive_small(b0 + 1);
        by0 = map_positive_small(b1) * 2654435761u;
        by1 = map_positive_small(b1 + 1) * 2654435761u;
        cz0 = map_positive_small(b2) * 805459861u;
        cz1 = map_positive_small(b2 + 1) * 805459861u;
    } else {
        const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                        b2 = static_cast<long long>(fl2);
        ax0 = map_positive32(b0);
        ax1 = map_positive32(b0 + 1);
        by0 = map_positive32(b1) * 2654435761u;
        by1 = map_positive32(b1 + 1) * 2654435761u;
        cz0 = map_positive32(b2) * 805459861u;
        cz1 = map_positive32(b2 + 1) * 805459861u;
    }
    if (T <= (1u << 28)) {
        // every row of the 16 levels indexes in 32 bits: (row & mask) | l T is one LOP3 and
        // the address one wide multiply-add (instead of a 64-bit slab add + shift per corner)
        const uint32_t lb = static_cast<uint32_t>(l) * T;
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
            const uint32_t rowi = ((ci & 1) ? ax1 : ax0) ^ ((ci & 2) ? by1 : by0) ^ ((ci & 4) ? cz1 : cz0);
            f.v[ci] = __ldg(tab + ((rowi & mask) | lb));
        }
    } else {
        const float2* slab = tab + static_cast<size_t>(l) * T;
#pragma unroll
        for (int ci = 0; ci < 8; ++ci) {
            const uint32_t rowi = ((ci & 1) ? ax1 : ax0) ^ ((ci & 2) ? by1 : by0) ^ ((ci & 4) ? cz1 : cz0);
            f.v[ci] = __ldg(slab + (rowi & mask));
        }
    }
    return f;
}

__device__ __forceinline__ float2 interp(const LevelFetch& f) {
    const float wx[2] = {1.0f - f.fr0, f.fr0}, wy[2] = {1.0f - f.fr1, f.fr1}, wz[2] = {1.0f - f.fr2, f.fr2};
    float g0 = 0.f, g1 = 0.f;
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {
        const float w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
        g0 += w * f.v[ci].x;
        g1 += w * f.v[ci].y;
    }
    return make_float2(g0 * f.dw, g1 * f.dw);
}

// Per level, what the backward's position / fade gradient needs from the gathered
// corners (hash_grid.hpp:104-121), so that the scatter does not gather the table again:
// o[0..1] = sum_c w_c T_c (the un-faded features), o[2 + 3 f + d] = sum_c (dw_c / dp_d) T_c,f
// (the trilinear Jacobian of feature f along lattice axis d).
__device__ __forceinline__ void level_sums(const LevelFetch& f, float* o) {
    const float wx[2] = {1.0f - f.fr0, f.fr0}, wy[2] = {1.0f - f.fr1, f.fr1}, wz[2] = {1.0f - f.fr2, f.fr2};
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.f;
#pragma unroll
    for (int ci = 0; ci < 8; ++ci) {
        const float ax = wx[ci & 1], ay = wy[(ci >> 1) & 1], az = wz[(ci >> 2) & 1];
        const float w = ax * ay * az;
        const float d0 = (ci & 1) ? ay * az : -(ay * az), d1 = (ci & 2) ? ax * az : -(ax * az),
                    d2 = (ci & 4) ? ax * ay : -(ax * ay);
        o[0] += w * f.v[ci].x;
        o[1] += w * f.v[ci].y;
        o[2] += d0 * f.v[ci].x;
        o[3] += d1 * f.v[ci].x;
        o[4] += d2 * f.v[ci].x;
        o[5] += d0 * f.v[ci].y;
        o[6] += d1 * f.v[ci].y;
        o[7] += d2 * f.v[ci].y;
    }
}

// The level fade alone (downweight, hash_grid.hpp:28-31), as fetch_level computes it.
__device__ __forceinline__ float level_fade(int l, const TcConst& cst, float ft, int no_downweight) {
    if (no_downweight) return 1.0f;
    const float r = ft * cst.inv_level_scale[l];
    return 1.0f - __expf(-r * r * 0.15915494309189535f);
}

// The lattice cell of one level without the gathers: the 8 corner rows (already
// masked to the table), the fractional position and the level fade. Used by the
// field backward, which scatters gradients to these rows.
struct LevelCell {
    uint32_t row[8];
    float fr0, fr1, fr2, dw;
};

template <bool kSmall>
__device__ __forceinline__ LevelCell level_cell(int l, double x0, double x1, double x2, const TcConst& cst,
                                                uint32_t mask, float ft, int no_downweight) {
    LevelCell c;
    const double s = cst.level_scale[l];
    const double p0 = s * x0, p1 = s * x1, p2 = s * x2;
    const double fl0 = floor(p0), fl1 = floor(p1), fl2 = floor(p2);
    c.fr0 = static_cast<float>(p0 - fl0);
    c.fr1 = static_cast<float>(p1 - fl1);
    c.fr2 = static_cast<float>(p2 - fl2);
    c.dw = 1.0f;
    if (!no_downweight) {
        const float r = ft * cst.inv_level_scale[l];
        c.dw = 1.0f - __expf(-r * r * 0.15915494309189535f);
    }
    uint32_t ax0, ax1, by0, by1, cz0, cz1;
    if (kSmall) {
        const int b0 = static_cast<int>(fl0), b1 = static_cast<int>(fl1), b2 = static_cast<int>(fl2);
        ax0 = map_positive_small(b0);
        ax1 = map_positive_small(b0 + 1);
        by0 = map_positive_small(b1) * 2654435761u;
        by1 = map_positive_small(b1 + 1) * 2654435761u;
        cz0 = map_positive_small(b2) * 805459861u;
        cz1 = map_positive_small(b2 + 1) * 805459861u;
    } else {
        const long long b0 = static_cast<long long>(fl0), b1 = static_cast<long long>(fl1),
                        b2 = static_cast<long long>(fl2);
        ax0 = map_positive32(b0);
        ax1 = map_positive32(b0 + 1);
        by0 = map_positive32(b1) * 2654435761u;
        by1 = map_positive32(b1 + 1) * 2654435761u;
        cz0 = map_positive32(b2) * 805459861u;
        cz1 = map_positive32(b2 + 1) * 805459861u;
    }
#pragma unroll
    for (int ci = 0; ci < 8; ++ci)
        c.row[ci] = (((ci & 1) ? ax1 : ax0) ^ ((ci & 2) ? by1 : by0) ^ ((ci & 4) ? cz1 : cz0)) & mask;
    return c;
}

}  // namespace
}  // namespace nx
