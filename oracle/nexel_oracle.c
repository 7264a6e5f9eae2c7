/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference render path (nexel::render =
 * collection_pass + texturing_pass) used as the parity checker for the CUDA
 * implementation. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. Scalar, single-threaded, fp64 throughout, with
 * each function citing the reference file:line it restates (paths relative to
 * /root/reference/proj/core/).
 *
 * Parity of this restatement is pinned against the reference itself: golden
 * fixtures produced by the reference compiled in place (oracle/_ref, recipe in
 * oracle/Makefile, fixtures by tests/golden/make_golden.py) — see
 * tests/test_oracle_golden.py.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/nexel_b200.h"

/* ---------------------------------------------------------------- vectors */
/* vec_math.hpp:9-67 */
typedef struct {
    double x, y, z;
} v3;

static v3 v3add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v3sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v3scale(double s, v3 a) { v3 r = {s * a.x, s * a.y, s * a.z}; return r; }
static double v3dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v3cross(v3 a, v3 b) {
    v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static double v3norm(v3 a) { return sqrt(v3dot(a, a)); }
/* normalized(a) = a / norm(a), per-component division (vec_math.hpp:35) */
static v3 v3normalized(v3 a) {
    double n = v3norm(a);
    v3 r = {a.x / n, a.y / n, a.z / n};
    return r;
}

static double sigmoid(double x) { /* vec_math.hpp:69-76 */
    if (x >= 0) {
        double e = exp(-x);
        return 1.0 / (1.0 + e);
    }
    double e = exp(x);
    return e / (1.0 + e);
}

static double softplus(double x) { /* vec_math.hpp:80-84 */
    if (x > 30.0) return x;
    if (x < -30.0) return exp(x);
    return log1p(exp(x));
}

/* ---------------------------------------------------------------- errors */
typedef struct {
    int status;
    char msg[256];
} orc_err;

static int fail(orc_err* e, int status, const char* msg) {
    if (e) {
        e->status = status;
        snprintf(e->msg, sizeof e->msg, "%s", msg);
    }
    return status;
}

static orc_err g_err;
const char* orc_last_error(void) { return g_err.msg; }

/* ---------------------------------------------------------------- settings + camera */
/* validate_settings, renderer.cpp:13-21 */
static int validate_settings(const nx_settings* s, orc_err* e) {
    if (s->top_k < 0 || s->top_k > NX_MAX_TOP_K) return fail(e, NX_BAD_SETTINGS, "top_k must be in [0, 8]");
    if (!(s->near_eps > 0)) return fail(e, NX_BAD_SETTINGS, "near_eps must be positive");
    if (!(s->alpha_max > 0) || s->alpha_max >= 1) return fail(e, NX_BAD_SETTINGS, "alpha_max must be in (0,1)");
    if (!(s->min_transmittance >= 0)) return fail(e, NX_BAD_SETTINGS, "min_transmittance must be >= 0");
    if (s->tile < 1) return fail(e, NX_BAD_SETTINGS, "tile must be >= 1");
    return NX_OK;
}

/* validate_camera, camera.cpp:8-31 */
static int validate_camera(const nx_camera* c, orc_err* e) {
    int i, j;
    if (c->width <= 0 || c->height <= 0) return fail(e, NX_BAD_CAMERA, "non-positive image size");
    if (!(c->fx > 0) || !(c->fy > 0)) return fail(e, NX_BAD_CAMERA, "non-positive focal length");
    for (i = 0; i < 3; ++i) {
        if (!isfinite(c->t[i])) return fail(e, NX_BAD_CAMERA, "non-finite translation");
        for (j = 0; j < 3; ++j)
            if (!isfinite(c->R[i * 3 + j])) return fail(e, NX_BAD_CAMERA, "non-finite rotation");
    }
    if (!isfinite(c->cx) || !isfinite(c->cy)) return fail(e, NX_BAD_CAMERA, "non-finite principal point");
    for (i = 0; i < 3; ++i)
        for (j = 0; j < 3; ++j) {
            double want = i == j ? 1.0 : 0.0;
            v3 ri = {c->R[i * 3], c->R[i * 3 + 1], c->R[i * 3 + 2]};
            v3 rj = {c->R[j * 3], c->R[j * 3 + 1], c->R[j * 3 + 2]};
            if (fabs(v3dot(ri, rj) - want) > 1e-9) return fail(e, NX_BAD_CAMERA, "rotation is not orthonormal");
        }
    {
        v3 r0 = {c->R[0], c->R[1], c->R[2]}, r1 = {c->R[3], c->R[4], c->R[5]}, r2 = {c->R[6], c->R[7], c->R[8]};
        if (v3dot(v3cross(r0, r1), r2) < 0) return fail(e, NX_BAD_CAMERA, "rotation is left-handed");
    }
    return NX_OK;
}

/* Camera (camera.hpp:17-43) */
static v3 cam_col(const nx_camera* c, int k) { v3 r = {c->R[k], c->R[3 + k], c->R[6 + k]}; return r; }
static v3 cam_row(const nx_camera* c, int k) { v3 r = {c->R[3 * k], c->R[3 * k + 1], c->R[3 * k + 2]}; return r; }
static v3 cam_t(const nx_camera* c) { v3 r = {c->t[0], c->t[1], c->t[2]}; return r; }
/* position() = -R^T t  (camera.hpp:24 via mul_transposed, vec_math.hpp:65-67) */
static v3 cam_position(const nx_camera* c) {
    v3 t = cam_t(c);
    v3 m = {v3dot(cam_col(c, 0), t), v3dot(cam_col(c, 1), t), v3dot(cam_col(c, 2), t)};
    v3 r = {-m.x, -m.y, -m.z};
    return r;
}
/* to_camera(p) = R p + t (camera.hpp:26) */
static v3 cam_to_camera(const nx_camera* c, v3 p) {
    v3 rp = {v3dot(cam_row(c, 0), p), v3dot(cam_row(c, 1), p), v3dot(cam_row(c, 2), p)};
    return v3add(rp, cam_t(c));
}
/* pixel_ray (camera.hpp:32-35) */
static void cam_pixel_ray(const nx_camera* c, double px, double py, v3* origin, v3* dir) {
    v3 d = {(px - c->cx) / c->fx, (py - c->cy) / c->fy, 1.0};
    v3 n = v3normalized(d);
    *origin = cam_position(c);
    dir->x = v3dot(cam_col(c, 0), n);
    dir->y = v3dot(cam_col(c, 1), n);
    dir->z = v3dot(cam_col(c, 2), n);
}
/* project (camera.hpp:38-42), min_depth 1e-9 */
static int cam_project(const nx_camera* c, v3 p, double* ox, double* oy) {
    v3 q = cam_to_camera(c, p);
    if (q.z < 1e-9) return 0;
    *ox = c->fx * q.x / q.z + c->cx;
    *oy = c->fy * q.y / q.z + c->cy;
    return 1;
}

/* ---------------------------------------------------------------- primitives */
/* ActivatedPrimitive (primitive.hpp:32-38) */
typedef struct {
    v3 mu;
    double R[3][3];
    double sx, sy, op, gx, gy;
} act_t;

static v3 act_col(const act_t* a, int k) { v3 r = {a->R[0][k], a->R[1][k], a->R[2][k]}; return r; }

/* quat_to_rotation (primitive.cpp:7-20), q = (w, x, y, z) */
static void quat_to_rotation(double w, double x, double y, double z, double R[3][3]) {
    R[0][0] = 1 - 2 * (y * y + z * z);
    R[0][1] = 2 * (x * y - w * z);
    R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z);
    R[1][1] = 1 - 2 * (x * x + z * z);
    R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y);
    R[2][1] = 2 * (y * z + w * x);
    R[2][2] = 1 - 2 * (x * x + y * y);
}

/* activate (primitive.cpp:47-76). p: 60 doubles in Nexel order. */
static int activate(const double* p, int64_t id, int gamma_frozen, act_t* a, orc_err* e) {
    int i;
    char buf[128];
    const char* what = NULL;
    for (i = 0; i < 3 && !what; ++i)
        if (!isfinite(p[i])) what = "non-finite position";
    for (i = 0; i < 4 && !what; ++i)
        if (!isfinite(p[3 + i])) what = "non-finite quaternion";
    for (i = 0; i < 2 && !what; ++i) {
        if (!isfinite(p[7 + i])) what = "non-finite log scale";
        else if (!isfinite(p[10 + i])) what = "non-finite kernel exponent";
    }
    if (!what && !isfinite(p[9])) what = "non-finite opacity";
    for (i = 0; i < NX_SH_VALUES && !what; ++i)
        if (!isfinite(p[12 + i])) what = "non-finite sh coefficient";
    if (!what) {
        double qn = sqrt(p[3] * p[3] + p[4] * p[4] + p[5] * p[5] + p[6] * p[6]);
        if (!(qn > 1e-12)) what = "degenerate quaternion";
        else {
            double s = 1.0 / qn;
            a->mu.x = p[0];
            a->mu.y = p[1];
            a->mu.z = p[2];
            quat_to_rotation(s * p[3], s * p[4], s * p[5], s * p[6], a->R);
            a->sx = exp(p[7]);
            a->sy = exp(p[8]);
            a->op = sigmoid(p[9]);
            if (gamma_frozen) {
                a->gx = 1.0;
                a->gy = 1.0;
            } else {
                a->gx = 1.0 + softplus(p[10]);
                a->gy = 1.0 + softplus(p[11]);
            }
            return NX_OK;
        }
    }
    snprintf(buf, sizeof buf, "%s in primitive %lld", what, (long long)id);
    return fail(e, NX_BAD_PRIMITIVE, buf);
}

/* ---------------------------------------------------------------- kernel */
#define K_ALPHA_MIN (1.0 / 255.0) /* kernel.hpp:11 */

static double axis_power(double u, double g) { /* kernel.hpp:16-22 */
    double e;
    if (u == 0.0) return 0.0;
    if (g == 1.0) return u * u;
    e = 2.0 * g * log(fabs(u));
    if (e > 700.0) return INFINITY;
    return exp(e);
}

static double eval_kernel(double u, double v, double o, double gx, double gy) { /* kernel.hpp:26-30 */
    double p = axis_power(u, gx) + axis_power(v, gy);
    if (isinf(p)) return 0.0;
    return o * exp(-0.5 * p);
}

static double support_radius(double o, double g) { /* kernel.hpp:72-76 */
    double lim = 2.0 * log(o / K_ALPHA_MIN);
    if (lim <= 0.0) return 0.0;
    return pow(lim, 1.0 / (2.0 * g));
}

/* intersect (intersect.hpp:23-42), kMinNormalDot = 1e-8 */
static int intersect(const act_t* a, v3 o, v3 d, double near_eps, double* t_out, double* alpha_out) {
    v3 n = act_col(a, 2);
    double denom = v3dot(d, n);
    double t, u, v, alpha;
    v3 delta;
    if (fabs(denom) < 1e-8) return 0;
    t = v3dot(v3sub(a->mu, o), n) / denom;
    if (!(t > near_eps)) return 0;
    delta = v3sub(v3add(o, v3scale(t, d)), a->mu);
    u = v3dot(delta, act_col(a, 0)) / a->sx;
    v = v3dot(delta, act_col(a, 1)) / a->sy;
    alpha = eval_kernel(u, v, a->op, a->gx, a->gy);
    if (alpha < K_ALPHA_MIN) return 0;
    *t_out = t;
    *alpha_out = alpha;
    return 1;
}

/* ---------------------------------------------------------------- SH */
/* sh_basis (sh.hpp:11-40) */
static void sh_basis(v3 d, double* b, int degree) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                          -1.0925484305920792, 0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                          0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                          -0.5900435899266435};
    double x = d.x, y = d.y, z = d.z, xx, yy, zz;
    b[0] = C0;
    if (degree < 1) return;
    b[1] = -C1 * y;
    b[2] = C1 * z;
    b[3] = -C1 * x;
    if (degree < 2) return;
    xx = x * x;
    yy = y * y;
    zz = z * z;
    b[4] = C2[0] * x * y;
    b[5] = C2[1] * y * z;
    b[6] = C2[2] * (2.0 * zz - xx - yy);
    b[7] = C2[3] * x * z;
    b[8] = C2[4] * (xx - yy);
    if (degree < 3) return;
    b[9] = C3[0] * y * (3.0 * xx - yy);
    b[10] = C3[1] * x * y * z;
    b[11] = C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = C3[5] * z * (xx - yy);
    b[15] = C3[6] * x * (xx - 3.0 * yy);
}

/* eval_sh (sh.hpp:46-57) */
static v3 eval_sh(const double* coeffs, v3 dir, int degree) {
    double b[16], rgb[3];
    int n = (degree + 1) * (degree + 1), c, k;
    v3 r;
    sh_basis(dir, b, degree);
    for (c = 0; c < 3; ++c) {
        double acc = 0.5;
        for (k = 0; k < n; ++k) acc += coeffs[k * 3 + c] * b[k];
        rgb[c] = acc < 0.0 ? 0.0 : acc;
    }
    r.x = rgb[0];
    r.y = rgb[1];
    r.z = rgb[2];
    return r;
}

/* ---------------------------------------------------------------- top-K */
/* TopKBuffer (framebuffers.hpp:14-57) */
typedef struct {
    int32_t id;
    double w, t;
    uint32_t seq;
} topk_e;
typedef struct {
    topk_e e[NX_MAX_TOP_K];
    int k, size;
    uint32_t counter;
} topk_t;

static void topk_reset(topk_t* b, int k) {
    int i;
    b->k = k;
    b->size = 0;
    b->counter = 0;
    for (i = 0; i < NX_MAX_TOP_K; ++i) {
        b->e[i].id = -1;
        b->e[i].w = 0;
        b->e[i].t = 0;
        b->e[i].seq = 0;
    }
}

static void topk_insert(topk_t* b, int32_t id, double w, double t) {
    uint32_t seq = b->counter++;
    int m = 0, i;
    if (b->size < b->k) {
        b->e[b->size].id = id;
        b->e[b->size].w = w;
        b->e[b->size].t = t;
        b->e[b->size].seq = seq;
        b->size++;
        return;
    }
    if (b->k == 0) return;
    for (i = 1; i < b->size; ++i)
        if (b->e[i].w < b->e[m].w || (b->e[i].w == b->e[m].w && b->e[i].seq > b->e[m].seq)) m = i;
    if (w > b->e[m].w) {
        b->e[m].id = id;
        b->e[m].w = w;
        b->e[m].t = t;
        b->e[m].seq = seq;
    }
}

/* finalize: weight desc, seq asc (insertion sort; framebuffers.hpp:51-56) */
static void topk_finalize(topk_t* b) {
    int i, j;
    for (i = 1; i < b->size; ++i) {
        topk_e x = b->e[i];
        j = i - 1;
        while (j >= 0 && (b->e[j].w < x.w || (b->e[j].w == x.w && b->e[j].seq > x.seq))) {
            b->e[j + 1] = b->e[j];
            --j;
        }
        b->e[j + 1] = x;
    }
}

/* ---------------------------------------------------------------- binning */
/* x86 cvttsd2si semantics for (int) of floor(...) results (out of range -> INT_MIN) */
static int to_int(double v) {
    if (v >= -2147483648.0 && v < 2147483648.0) return (int)v;
    return INT32_MIN;
}
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

typedef struct {
    double depth;
    int32_t id;
    int tx0, tx1, ty0, ty1;
} entry_t;

static int entry_cmp(const void* pa, const void* pb) { /* renderer.cpp:102-105 */
    const entry_t* a = (const entry_t*)pa;
    const entry_t* b = (const entry_t*)pb;
    if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

typedef struct {
    act_t* act;
    int tiles_x, tiles_y;
    int64_t* offsets; /* n_tiles + 1 */
    int32_t* ids;     /* P */
    int64_t n_entries, n_straddlers;
} binning_t;

static void binning_free(binning_t* b) {
    free(b->act);
    free(b->offsets);
    free(b->ids);
    memset(b, 0, sizeof *b);
}

/* build_binning (renderer.cpp:36-111) */
static int build_binning(const nx_settings* st, int64_t n, const double* nexels, const nx_camera* cam,
                         binning_t* bin, orc_err* e) {
    const int tile = st->tile;
    int64_t i, ne = 0, t, n_tiles;
    entry_t* entries;
    int64_t* fill;
    memset(bin, 0, sizeof *bin);
    bin->act = (act_t*)malloc(sizeof(act_t) * (size_t)(n > 0 ? n : 1));
    for (i = 0; i < n; ++i) {
        int s = activate(nexels + i * NX_PARAMS_PER_NEXEL, i, st->no_gamma, &bin->act[i], e);
        if (s) {
            free(bin->act);
            bin->act = NULL;
            return s;
        }
    }
    bin->tiles_x = (cam->width + tile - 1) / tile;
    bin->tiles_y = (cam->height + tile - 1) / tile;
    n_tiles = (int64_t)bin->tiles_x * bin->tiles_y;
    entries = (entry_t*)malloc(sizeof(entry_t) * (size_t)(n > 0 ? n : 1));
    for (i = 0; i < n; ++i) {
        const act_t* a = &bin->act[i];
        double ru = support_radius(a->op, a->gx), rv = support_radius(a->op, a->gy);
        v3 du, dv, corners[4];
        int all_behind, all_visible = 1, c;
        double px0 = 1e300, px1 = -1e300, py0 = 1e300, py1 = -1e300;
        entry_t en;
        if (ru <= 0.0 || rv <= 0.0) continue;
        du = v3scale(ru * a->sx, act_col(a, 0));
        dv = v3scale(rv * a->sy, act_col(a, 1));
        corners[0] = v3add(v3add(a->mu, du), dv);
        corners[1] = v3sub(v3add(a->mu, du), dv);
        corners[2] = v3add(v3sub(a->mu, du), dv);
        corners[3] = v3sub(v3sub(a->mu, du), dv);
        all_behind = cam_to_camera(cam, a->mu).z < 1e-9;
        for (c = 0; c < 4; ++c) {
            double x, y;
            if (!cam_project(cam, corners[c], &x, &y)) {
                all_visible = 0;
                continue;
            }
            all_behind = 0;
            px0 = fmin(px0, x); /* std::min/max on non-NaN values */
            px1 = fmax(px1, x);
            py0 = fmin(py0, y);
            py1 = fmax(py1, y);
        }
        if (all_behind && !all_visible) continue;
        en.depth = cam_to_camera(cam, a->mu).z;
        en.id = (int32_t)i;
        if (all_visible) {
            int ix0 = to_int(floor(px0 - 1.5)), ix1 = to_int(ceil(px1 + 0.5));
            int iy0 = to_int(floor(py0 - 1.5)), iy1 = to_int(ceil(py1 + 0.5));
            if (ix1 < 0 || iy1 < 0 || ix0 >= cam->width || iy0 >= cam->height) continue;
            en.tx0 = clampi(ix0, 0, cam->width - 1) / tile;
            en.tx1 = clampi(ix1, 0, cam->width - 1) / tile;
            en.ty0 = clampi(iy0, 0, cam->height - 1) / tile;
            en.ty1 = clampi(iy1, 0, cam->height - 1) / tile;
        } else {
            en.tx0 = 0;
            en.tx1 = bin->tiles_x - 1;
            en.ty0 = 0;
            en.ty1 = bin->tiles_y - 1;
            bin->n_straddlers++;
        }
        entries[ne++] = en;
    }
    bin->n_entries = ne;
    qsort(entries, (size_t)ne, sizeof(entry_t), entry_cmp);
    bin->offsets = (int64_t*)calloc((size_t)n_tiles + 1, sizeof(int64_t));
    for (i = 0; i < ne; ++i) {
        int tx, ty;
        for (ty = entries[i].ty0; ty <= entries[i].ty1; ++ty)
            for (tx = entries[i].tx0; tx <= entries[i].tx1; ++tx) bin->offsets[(int64_t)ty * bin->tiles_x + tx + 1]++;
    }
    for (t = 0; t < n_tiles; ++t) bin->offsets[t + 1] += bin->offsets[t];
    bin->ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(bin->offsets[n_tiles] > 0 ? bin->offsets[n_tiles] : 1));
    fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_tiles);
    memcpy(fill, bin->offsets, sizeof(int64_t) * (size_t)n_tiles);
    for (i = 0; i < ne; ++i) {
        int tx, ty;
        for (ty = entries[i].ty0; ty <= entries[i].ty1; ++ty)
            for (tx = entries[i].tx0; tx <= entries[i].tx1; ++tx)
                bin->ids[fill[(int64_t)ty * bin->tiles_x + tx]++] = entries[i].id;
    }
    free(fill);
    free(entries);
    return NX_OK;
}

/* ---------------------------------------------------------------- hash grid + MLP */
static uint64_t map_positive(int64_t x) { /* hash_grid.hpp:12-14 */
    return x > 0 ? (uint64_t)(2 * x - 1) : (uint64_t)(-2 * x);
}
static uint32_t hash_cell(int64_t ix, int64_t iy, int64_t iz, uint32_t T) { /* hash_grid.hpp:17-23 */
    uint32_t a = (uint32_t)map_positive(ix);
    uint32_t b = (uint32_t)map_positive(iy) * 2654435761u;
    uint32_t c = (uint32_t)map_positive(iz) * 805459861u;
    return (a ^ b ^ c) & (T - 1);
}
static double downweight(double s, double t, double f) { /* hash_grid.hpp:28-31 */
    double r = f / (s * t);
    return 1.0 - exp(-r * r / (2.0 * M_PI));
}

typedef struct {
    const nx_field_desc* d;
    const double *table, *w1, *w2, *w3;
} field_t;

/* grid_lookup (hash_grid.cpp:26-83) */
static void grid_lookup(const field_t* f, v3 x, double t, double fl, double* out, int no_downweight) {
    const int F = f->d->features;
    const uint32_t T = 1u << f->d->log2_table;
    double s = f->d->base_scale;
    int l, ci, fi;
    for (l = 0; l < f->d->levels; ++l, s *= f->d->growth) {
        v3 p = v3scale(s, x);
        double fx = floor(p.x), fy = floor(p.y), fz = floor(p.z);
        int64_t bx = (int64_t)fx, by = (int64_t)fy, bz = (int64_t)fz;
        double frx = p.x - fx, fry = p.y - fy, frz = p.z - fz;
        double dw = no_downweight ? 1.0 : downweight(s, t, fl);
        double wx[2] = {1.0 - frx, frx}, wy[2] = {1.0 - fry, fry}, wz[2] = {1.0 - frz, frz};
        double* g = out + (size_t)l * F;
        size_t slab = (size_t)l * T;
        for (fi = 0; fi < F; ++fi) g[fi] = 0.0;
        for (ci = 0; ci < 8; ++ci) {
            uint32_t row = hash_cell(bx + (ci & 1), by + ((ci >> 1) & 1), bz + ((ci >> 2) & 1), T);
            double w = wx[ci & 1] * wy[(ci >> 1) & 1] * wz[(ci >> 2) & 1];
            const double* feat = f->table + (slab + row) * F;
            for (fi = 0; fi < F; ++fi) g[fi] += w * feat[fi];
        }
        for (fi = 0; fi < F; ++fi) g[fi] *= dw;
    }
}

/* TextureMlp::forward (mlp.cpp:24-43), bias-free ReLU MLP, row-major [out][in] */
static void mlp_forward(const field_t* f, const double* x, double* y) {
    const int nin = f->d->levels * f->d->features, nh = f->d->n_hidden, nout = NX_SH_VALUES;
    double h1[256], h2[256];
    int o, i;
    for (o = 0; o < nh; ++o) {
        double acc = 0.0;
        for (i = 0; i < nin; ++i) acc += f->w1[(size_t)o * nin + i] * x[i];
        h1[o] = acc > 0.0 ? acc : 0.0;
    }
    for (o = 0; o < nh; ++o) {
        double acc = 0.0;
        for (i = 0; i < nh; ++i) acc += f->w2[(size_t)o * nh + i] * h1[i];
        h2[o] = acc > 0.0 ? acc : 0.0;
    }
    for (o = 0; o < nout; ++o) {
        double acc = 0.0;
        for (i = 0; i < nh; ++i) acc += f->w3[(size_t)o * nh + i] * h2[i];
        y[o] = acc;
    }
}

/* field_forward (texture_field.cpp:20-31): lookup -> MLP -> eval_sh(coeffs, dir, 3) */
static v3 field_forward(const field_t* f, v3 x, double t, double fl, v3 dir, int no_downweight) {
    double feats[256], coeffs[NX_SH_VALUES];
    grid_lookup(f, x, t, fl, feats, no_downweight);
    mlp_forward(f, feats, coeffs);
    return eval_sh(coeffs, dir, 3);
}

/* ---------------------------------------------------------------- entry points */
typedef struct orc_stats {
    int64_t n_entries, n_straddlers, tile_keys, n_queries, n_tests, n_hits;
} orc_stats;

static int check_field(const nx_field_desc* d, orc_err* e) {
    if (d->levels < 1 || d->features < 1 || d->levels * d->features > 256 || d->n_hidden < 1 ||
        d->n_hidden > 256 || d->log2_table < 0 || d->log2_table > 30)
        return fail(e, NX_UNSUPPORTED, "field shape outside the oracle's limits");
    return NX_OK;
}

/*
 * render (renderer.cpp:239-244) = collection_pass (renderer.cpp:115-171) +
 * texturing_pass (renderer.cpp:207-237, build_queries renderer.cpp:177-203).
 * Outputs are FrameBuffers-shaped doubles (ids int32); NULL outputs are skipped
 * except that ids/depths/weights/base are needed internally (allocated if NULL).
 */
int orc_render(const nx_settings* st, int64_t n, const double* nexels, const nx_field_desc* fd,
               const double* table, const double* w1, const double* w2, const double* w3,
               const nx_camera* cam, double* base, int32_t* ids, double* depths, double* weights,
               double* texture, double* final_img, double* residual, orc_stats* stats) {
    orc_err* e = &g_err;
    binning_t bin;
    field_t field = {fd, table, w1, w2, w3};
    const int K = st->top_k, tile = st->tile, degree = st->no_prim_sh ? 0 : 3;
    int64_t W, H, npix, p, t, n_tiles, q = 0, tests = 0, hits = 0;
    int s;
    double *b_ = base, *d_ = depths, *w_ = weights, *r_ = residual;
    int32_t* i_ = ids;
    v3 bg = {st->background[0], st->background[1], st->background[2]};

    e->status = 0;
    e->msg[0] = 0;
    if ((s = validate_settings(st, e))) return s;
    if ((s = validate_camera(cam, e))) return s;
    if ((s = check_field(fd, e))) return s;
    W = cam->width;
    H = cam->height;
    npix = W * H;
    if ((s = build_binning(st, n, nexels, cam, &bin, e))) return s;
    n_tiles = (int64_t)bin.tiles_x * bin.tiles_y;

    /* FrameBuffers::allocate (framebuffers.hpp:71-82) */
    if (!b_) b_ = (double*)malloc(sizeof(double) * (size_t)(npix * 3));
    if (!i_) i_ = (int32_t*)malloc(sizeof(int32_t) * (size_t)(npix * K + 1));
    if (!d_) d_ = (double*)malloc(sizeof(double) * (size_t)(npix * K + 1));
    if (!w_) w_ = (double*)malloc(sizeof(double) * (size_t)(npix * K + 1));
    if (!r_) r_ = (double*)malloc(sizeof(double) * (size_t)npix);
    for (p = 0; p < npix * K; ++p) {
        i_[p] = -1;
        d_[p] = 0.0;
        w_[p] = 0.0;
        if (texture) texture[3 * p] = texture[3 * p + 1] = texture[3 * p + 2] = 0.0;
    }

    /* collection_pass: per tile, per pixel march (renderer.cpp:129-169) */
    for (t = 0; t < n_tiles; ++t) {
        const int ty = (int)(t / bin.tiles_x), tx = (int)(t % bin.tiles_x);
        const int x1 = (int)(W < (tx + 1) * tile ? W : (tx + 1) * tile);
        const int y1 = (int)(H < (ty + 1) * tile ? H : (ty + 1) * tile);
        int px, py, j;
        for (py = ty * tile; py < y1; ++py)
            for (px = tx * tile; px < x1; ++px) {
                v3 o, d, acc = {0, 0, 0};
                double T = 1.0;
                int64_t pix = (int64_t)py * W + px, li;
                topk_t tk;
                cam_pixel_ray(cam, px + 0.5, py + 0.5, &o, &d);
                topk_reset(&tk, K);
                for (li = bin.offsets[t]; li < bin.offsets[t + 1]; ++li) {
                    const int32_t id = bin.ids[li];
                    double th, ah, alpha, w;
                    ++tests;
                    if (!intersect(&bin.act[id], o, d, st->near_eps, &th, &ah)) continue;
                    ++hits;
                    alpha = ah < st->alpha_max ? ah : st->alpha_max; /* std::min */
                    w = alpha * T;
                    acc = v3add(acc, v3scale(w, eval_sh(nexels + (int64_t)id * NX_PARAMS_PER_NEXEL + 12, d, degree)));
                    topk_insert(&tk, id, w, th);
                    T *= 1.0 - alpha;
                    if (T < st->min_transmittance) break;
                }
                r_[pix] = T;
                acc = v3add(acc, v3scale(T, bg));
                topk_finalize(&tk);
                for (j = 0; j < tk.size; ++j) {
                    int64_t sl = pix * K + j;
                    i_[sl] = tk.e[j].id;
                    d_[sl] = tk.e[j].t;
                    w_[sl] = tk.e[j].w;
                    acc = v3sub(acc, v3scale(tk.e[j].w, eval_sh(nexels + (int64_t)tk.e[j].id * NX_PARAMS_PER_NEXEL + 12, d, degree)));
                }
                b_[pix * 3 + 0] = acc.x;
                b_[pix * 3 + 1] = acc.y;
                b_[pix * 3 + 2] = acc.z;
            }
    }

    /* texturing_pass: queries pixel-major, slot-minor (renderer.cpp:177-203), then
     * final = base + sum_j W[p,j] T[p,j] (renderer.cpp:219-236). */
    for (p = 0; p < npix; ++p) {
        v3 acc = {b_[p * 3], b_[p * 3 + 1], b_[p * 3 + 2]};
        int j;
        if (K > 0) {
            v3 o, d;
            int have = 0;
            for (j = 0; j < K; ++j) {
                int64_t sl = p * K + j;
                v3 x, rgb;
                double w;
                if (i_[sl] < 0) continue;
                if (!have) {
                    cam_pixel_ray(cam, (double)(p % W) + 0.5, (double)(p / W) + 0.5, &o, &d);
                    have = 1;
                }
                x = v3add(o, v3scale(d_[sl], d));
                rgb = field_forward(&field, x, d_[sl], cam->fx, d, st->no_downweight);
                ++q;
                if (texture) {
                    texture[sl * 3 + 0] = rgb.x;
                    texture[sl * 3 + 1] = rgb.y;
                    texture[sl * 3 + 2] = rgb.z;
                }
                w = w_[sl];
                acc.x += w * rgb.x;
                acc.y += w * rgb.y;
                acc.z += w * rgb.z;
            }
        }
        if (final_img) {
            final_img[p * 3 + 0] = acc.x;
            final_img[p * 3 + 1] = acc.y;
            final_img[p * 3 + 2] = acc.z;
        }
    }

    if (stats) {
        stats->n_entries = bin.n_entries;
        stats->n_straddlers = bin.n_straddlers;
        stats->tile_keys = bin.offsets[n_tiles];
        stats->n_queries = q;
        stats->n_tests = tests;
        stats->n_hits = hits;
    }
    if (b_ != base) free(b_);
    if (i_ != ids) free(i_);
    if (d_ != depths) free(d_);
    if (w_ != weights) free(w_);
    if (r_ != residual) free(r_);
    binning_free(&bin);
    return NX_OK;
}

/* Binning::tile_lists as CSR (renderer.cpp:102-110). */
int orc_tile_lists(const nx_settings* st, int64_t n, const double* nexels, const nx_camera* cam,
                   int64_t* offsets, int32_t* ids, int64_t capacity, int64_t* total, int32_t* tiles_x,
                   int32_t* tiles_y) {
    orc_err* e = &g_err;
    binning_t bin;
    int64_t nt, i;
    int s;
    if ((s = validate_settings(st, e))) return s;
    if ((s = validate_camera(cam, e))) return s;
    if ((s = build_binning(st, n, nexels, cam, &bin, e))) return s;
    nt = (int64_t)bin.tiles_x * bin.tiles_y;
    *tiles_x = bin.tiles_x;
    *tiles_y = bin.tiles_y;
    *total = bin.offsets[nt];
    if (offsets) memcpy(offsets, bin.offsets, sizeof(int64_t) * (size_t)(nt + 1));
    if (ids)
        for (i = 0; i < bin.offsets[nt] && i < capacity; ++i) ids[i] = bin.ids[i];
    binning_free(&bin);
    return NX_OK;
}

/* Per-pixel contributor sequences for rows [y0,y1): the collection march
 * (renderer.cpp:137-153) recording hit ids up to termination. */
int orc_pixel_hits(const nx_settings* st, int64_t n, const double* nexels, const nx_camera* cam, int y0,
                   int y1, int max_hits, int32_t* hits, int32_t* counts) {
    orc_err* e = &g_err;
    binning_t bin;
    int s, py, px;
    if ((s = validate_settings(st, e))) return s;
    if ((s = validate_camera(cam, e))) return s;
    if ((s = build_binning(st, n, nexels, cam, &bin, e))) return s;
    for (py = y0; py < y1; ++py)
        for (px = 0; px < cam->width; ++px) {
            int64_t q = (int64_t)(py - y0) * cam->width + px;
            int64_t t = (int64_t)(py / st->tile) * bin.tiles_x + px / st->tile, li;
            v3 o, d;
            double T = 1.0;
            int cnt = 0;
            cam_pixel_ray(cam, px + 0.5, py + 0.5, &o, &d);
            for (li = bin.offsets[t]; li < bin.offsets[t + 1]; ++li) {
                double th, ah, alpha;
                int32_t id = bin.ids[li];
                if (!intersect(&bin.act[id], o, d, st->near_eps, &th, &ah)) continue;
                if (cnt < max_hits) hits[q * max_hits + cnt] = id;
                ++cnt;
                alpha = ah < st->alpha_max ? ah : st->alpha_max;
                T *= 1.0 - alpha;
                if (T < st->min_transmittance) break;
            }
            counts[q] = cnt;
        }
    binning_free(&bin);
    return NX_OK;
}

/* Known-answer hooks (geometry + field), for tests against the reference values. */
double orc_eval_kernel(double u, double v, double o, double gx, double gy) { return eval_kernel(u, v, o, gx, gy); }
double orc_support_radius(double o, double g) { return support_radius(o, g); }
uint32_t orc_hash_cell(int64_t ix, int64_t iy, int64_t iz, uint32_t T) { return hash_cell(ix, iy, iz, T); }
uint64_t orc_map_positive(int64_t x) { return map_positive(x); }
double orc_downweight(double s, double t, double f) { return downweight(s, t, f); }
void orc_sh_basis(const double* dir, double* b) {
    v3 d = {dir[0], dir[1], dir[2]};
    sh_basis(d, b, 3);
}
/* TopKBuffer round trip: inserts (ids, w, t) then finalize; writes size + slots. */
int orc_topk(int k, int n, const int32_t* ids, const double* w, const double* t, int32_t* out_ids, double* out_w) {
    topk_t b;
    int i;
    topk_reset(&b, k);
    for (i = 0; i < n; ++i) topk_insert(&b, ids[i], w[i], t[i]);
    topk_finalize(&b);
    for (i = 0; i < k; ++i) {
        out_ids[i] = b.e[i].id;
        out_w[i] = b.e[i].w;
    }
    return b.size;
}
int orc_field_forward(const nx_field_desc* fd, const double* table, const double* w1, const double* w2,
                      const double* w3, int64_t n, const double* q8, int no_downweight, double* rgb) {
    field_t field = {fd, table, w1, w2, w3};
    int64_t i;
    if (check_field(fd, &g_err)) return NX_UNSUPPORTED;
    for (i = 0; i < n; ++i) {
        const double* r = q8 + i * 8;
        v3 x = {r[0], r[1], r[2]}, dir = {r[5], r[6], r[7]};
        v3 c = field_forward(&field, x, r[3], r[4], dir, no_downweight);
        rgb[i * 3] = c.x;
        rgb[i * 3 + 1] = c.y;
        rgb[i * 3 + 2] = c.z;
    }
    return NX_OK;
}
