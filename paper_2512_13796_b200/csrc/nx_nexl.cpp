// NEXL checkpoint reader (checkpoint.cpp:52-97 Reader, :173-271 load_checkpoint): the
// host side of nx_scene_load_nexl / nx_nexl_cameras. Little-endian fields, learnable
// arrays fp32, config and cameras fp64 — parsed with the reference's checks and
// messages, the fp32 sections read in bulk (no per-value conversion on the host).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nexel_b200.h"
#include "nx_nexl.h"

namespace nx {

namespace {

struct Reader {
    FILE* f = nullptr;
    std::string path;
    int status = NX_OK;
    std::string msg;

    explicit Reader(const char* p) : path(p ? p : "") {
        f = p ? std::fopen(p, "rb") : nullptr;
        if (!f) fail(NX_MISSING_FILE, "cannot open " + path);
    }
    ~Reader() {
        if (f) std::fclose(f);
    }
    bool ok() const { return status == NX_OK; }
    void fail(int st, const std::string& m) {
        if (status == NX_OK) {
            status = st;
            msg = m;
        }
    }
    void bytes(void* p, size_t n) {
        if (!ok()) {
            std::memset(p, 0, n);
            return;
        }
        if (std::fread(p, 1, n, f) != n) {
            std::memset(p, 0, n);
            fail(NX_BAD_CHECKPOINT, path + ": truncated");
        }
    }
    uint32_t u32() {
        unsigned char b[4];
        bytes(b, 4);
        return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
    }
    uint64_t u64() {
        const uint64_t lo = u32();
        return lo | (uint64_t(u32()) << 32);
    }
    int64_t i64() { return static_cast<int64_t>(u64()); }
    double f64() {
        const uint64_t v = u64();
        double d;
        std::memcpy(&d, &v, 8);
        return d;
    }
    std::string str() {
        const uint32_t n = u32();
        if (n > (1u << 20)) {
            fail(NX_BAD_CHECKPOINT, path + ": absurd string length");
            return {};
        }
        std::string s(n, '\0');
        bytes(s.data(), n);
        return s;
    }
    void skip(uint64_t n) {
        if (ok() && std::fseek(f, static_cast<long>(n), SEEK_CUR) != 0) fail(NX_BAD_CHECKPOINT, path + ": truncated");
    }
    // little-endian fp32 array (the host is little-endian x86-64)
    void f32s(float* p, size_t n) { bytes(p, n * sizeof(float)); }
};

int read_header(Reader& r, NexlHeader& h) {
    char magic[4];
    r.bytes(magic, 4);
    if (r.ok() && std::memcmp(magic, "NEXL", 4) != 0) r.fail(NX_BAD_CHECKPOINT, r.path + ": wrong magic");
    const uint32_t version = r.u32();
    if (r.ok() && version != 1) r.fail(NX_BAD_CHECKPOINT, r.path + ": unsupported version " + std::to_string(version));
    const uint32_t flags = r.u32();
    nx_settings_default(&h.info.settings);
    nx_settings& rs = h.info.settings;
    rs.no_gamma = (flags >> 1) & 1;
    rs.no_prim_sh = (flags >> 2) & 1;
    rs.no_downweight = (flags >> 3) & 1;
    h.info.has_optimizer = flags & 1;
    rs.top_k = static_cast<int32_t>(r.u32());
    for (int c = 0; c < 3; ++c) rs.background[c] = r.f64();
    rs.near_eps = r.f64();
    rs.alpha_max = r.f64();
    rs.min_transmittance = r.f64();
    rs.tile = static_cast<int32_t>(r.u32());
    h.info.extent = r.f64();
    h.info.iteration = r.u64();
    nx_field_desc& fd = h.info.field;
    fd.levels = static_cast<int32_t>(r.u32());
    fd.log2_table = static_cast<int32_t>(r.u32());
    fd.features = static_cast<int32_t>(r.u32());
    fd.base_scale = r.f64();
    fd.growth = r.f64();
    if (r.ok() && (fd.levels <= 0 || fd.levels > 64 || fd.log2_table <= 0 || fd.log2_table > 26 || fd.features <= 0 ||
                   fd.features > 16))
        r.fail(NX_BAD_CHECKPOINT, r.path + ": implausible grid shape");
    const uint32_t n_in = r.u32();
    fd.n_hidden = static_cast<int32_t>(r.u32());
    const uint32_t n_out = r.u32();
    if (r.ok() && (static_cast<int>(n_in) != fd.levels * fd.features || n_out != NX_SH_VALUES || fd.n_hidden <= 0 ||
                   fd.n_hidden > 4096))
        r.fail(NX_BAD_CHECKPOINT, r.path + ": implausible mlp shape");
    const uint32_t n_cams = r.u32();
    if (r.ok() && n_cams > (1u << 20)) r.fail(NX_BAD_CHECKPOINT, r.path + ": absurd camera count");
    if (!r.ok()) return r.status;
    h.info.n_cameras = static_cast<int32_t>(n_cams);
    h.cameras.resize(n_cams);
    h.names.resize(n_cams);
    for (uint32_t i = 0; i < n_cams && r.ok(); ++i) {
        nx_camera& c = h.cameras[i];
        h.names[i] = r.str();
        c.width = static_cast<int32_t>(r.u32());
        c.height = static_cast<int32_t>(r.u32());
        c.fx = r.f64();
        c.fy = r.f64();
        c.cx = r.f64();
        c.cy = r.f64();
        for (int k = 0; k < 9; ++k) c.R[k] = r.f64();
        for (int k = 0; k < 3; ++k) c.t[k] = r.f64();
    }
    const uint64_t n = r.u64();
    if (r.ok() && n > (1ull << 32)) r.fail(NX_BAD_CHECKPOINT, r.path + ": absurd primitive count");
    h.info.n_nexels = static_cast<int64_t>(n);
    return r.status;
}

}  // namespace

int nexl_read(const char* path, bool with_arrays, NexlHeader& h, NexlArrays* arr, std::string& err) {
    Reader r(path);
    int st = r.ok() ? read_header(r, h) : r.status;
    if (st) {
        err = r.msg;
        return st;
    }
    if (with_arrays && arr) {
        const size_t n = static_cast<size_t>(h.info.n_nexels);
        const nx_field_desc& fd = h.info.field;
        const size_t n_in = static_cast<size_t>(fd.levels) * fd.features, nh = fd.n_hidden;
        try {
            arr->mu.resize(n * 3);
            arr->quat.resize(n * 4);
            arr->log_scale.resize(n * 2);
            arr->opacity.resize(n);
            arr->gamma.resize(n * 2);
            arr->sh.resize(n * NX_SH_VALUES);
            arr->table.resize(static_cast<size_t>(fd.levels) * (size_t(1) << fd.log2_table) * fd.features);
            arr->w1.resize(nh * n_in);
            arr->w2.resize(nh * nh);
            arr->w3.resize(NX_SH_VALUES * nh);
        } catch (const std::bad_alloc&) {
            err = "host allocation";
            return NX_OUT_OF_MEMORY;
        }
        r.f32s(arr->mu.data(), arr->mu.size());
        r.f32s(arr->quat.data(), arr->quat.size());
        r.f32s(arr->log_scale.data(), arr->log_scale.size());
        r.f32s(arr->opacity.data(), arr->opacity.size());
        r.f32s(arr->gamma.data(), arr->gamma.size());
        r.f32s(arr->sh.data(), arr->sh.size());
        r.f32s(arr->table.data(), arr->table.size());
        r.f32s(arr->w1.data(), arr->w1.size());
        r.f32s(arr->w2.data(), arr->w2.size());
        r.f32s(arr->w3.data(), arr->w3.size());
        // the optimizer section (if any) is not part of a render scene
    }
    if (!r.ok()) err = r.msg;
    return r.status;
}

}  // namespace nx

extern "C" int nx_nexl_cameras(const char* path, nx_camera* cams, char (*names)[64], int capacity, int* n) {
    nx::NexlHeader h;
    std::string err;
    const int st = nx::nexl_read(path, false, h, nullptr, err);
    if (st) return st;
    if (n) *n = h.info.n_cameras;
    for (int i = 0; i < h.info.n_cameras && i < capacity; ++i) {
        if (cams) cams[i] = h.cameras[i];
        if (names) {
            std::strncpy(names[i], h.names[i].c_str(), 63);
            names[i][63] = '\0';
        }
    }
    return NX_OK;
}
