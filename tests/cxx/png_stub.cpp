// Test-only stand-in for the reference's image.cpp (which needs libpng, absent from
// this image): nexel::save_png / load_png for 8-bit RGB PNGs whose zlib stream uses
// stored (uncompressed) deflate blocks — enough for the synthetic bundles the
// reference's own tests write and read back (test_train.cpp tiny_bundle via
// make_synthetic_bundle + load_bundle). Quantisation as the reference's writer:
// byte = lround(clamp01(x) * 255), read back as byte / 255.
#include "nexel/image.hpp"

#include <cmath>
#include <cstdint>
#include <fstream>
#include <string>
#include <vector>

#include "nexel/error.hpp"

namespace nexel {

namespace {

uint32_t crc32(const uint8_t* p, size_t n, uint32_t c = 0xffffffffu) {
    for (size_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xedb88320u & (0u - (c & 1u)));
    }
    return c;
}

void put32(std::vector<uint8_t>& o, uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) o.push_back(static_cast<uint8_t>(v >> s));
}

uint32_t get32(const uint8_t* p) {
    return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}

void chunk(std::vector<uint8_t>& o, const char* type, const std::vector<uint8_t>& data) {
    put32(o, static_cast<uint32_t>(data.size()));
    std::vector<uint8_t> td(type, type + 4);
    td.insert(td.end(), data.begin(), data.end());
    o.insert(o.end(), td.begin(), td.end());
    put32(o, crc32(td.data(), td.size()) ^ 0xffffffffu);
}

const uint8_t kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

}  // namespace

void save_png(const std::string& path, const Image& img) {
    const int w = img.width, h = img.height;
    std::vector<uint8_t> raw;
    raw.reserve(static_cast<size_t>(h) * (1 + 3 * w));
    for (int y = 0; y < h; ++y) {
        raw.push_back(0);  // filter: none
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < 3; ++c) {
                const double v = std::min(1.0, std::max(0.0, img.px[(static_cast<size_t>(y) * w + x) * 3 + c]));
                raw.push_back(static_cast<uint8_t>(std::lround(v * 255.0)));
            }
    }
    std::vector<uint8_t> z = {0x78, 0x01};
    uint32_t a = 1, b = 0;
    for (uint8_t v : raw) {
        a = (a + v) % 65521u;
        b = (b + a) % 65521u;
    }
    size_t pos = 0;
    do {
        const size_t len = std::min<size_t>(65535, raw.size() - pos);
        z.push_back(pos + len == raw.size() ? 1 : 0);
        z.push_back(static_cast<uint8_t>(len));
        z.push_back(static_cast<uint8_t>(len >> 8));
        z.push_back(static_cast<uint8_t>(~len));
        z.push_back(static_cast<uint8_t>(~len >> 8));
        z.insert(z.end(), raw.begin() + pos, raw.begin() + pos + len);
        pos += len;
    } while (pos < raw.size());
    put32(z, (b << 16) | a);
    std::vector<uint8_t> o(kSig, kSig + 8), ihdr;
    put32(ihdr, static_cast<uint32_t>(w));
    put32(ihdr, static_cast<uint32_t>(h));
    ihdr.insert(ihdr.end(), {8, 2, 0, 0, 0});
    chunk(o, "IHDR", ihdr);
    chunk(o, "IDAT", z);
    chunk(o, "IEND", {});
    std::ofstream f(path, std::ios::binary);
    if (!f) fail("io-error", "cannot write " + path);
    f.write(reinterpret_cast<const char*>(o.data()), static_cast<std::streamsize>(o.size()));
}

Image load_png(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) fail("missing-file", "cannot open " + path);
    std::vector<uint8_t> d((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (d.size() < 8 || !std::equal(kSig, kSig + 8, d.begin())) fail("bad-image", path + ": not a PNG");
    int w = 0, h = 0;
    std::vector<uint8_t> z;
    for (size_t p = 8; p + 12 <= d.size();) {
        const uint32_t len = get32(&d[p]);
        const std::string type(d.begin() + p + 4, d.begin() + p + 8);
        const uint8_t* data = &d[p + 8];
        if (type == "IHDR") {
            w = static_cast<int>(get32(data));
            h = static_cast<int>(get32(data + 4));
            if (data[8] != 8 || data[9] != 2 || data[12] != 0) fail("bad-image", path + ": only 8-bit RGB stubbed");
        } else if (type == "IDAT") {
            z.insert(z.end(), data, data + len);
        }
        p += 12 + len;
    }
    std::vector<uint8_t> raw;
    for (size_t p = 2; p < z.size();) {  // stored deflate blocks only
        const uint8_t hdr = z[p];
        if ((hdr >> 1) & 3) fail("bad-image", path + ": compressed PNG data is not stubbed");
        const size_t len = z[p + 1] | (size_t(z[p + 2]) << 8);
        raw.insert(raw.end(), z.begin() + p + 5, z.begin() + p + 5 + len);
        p += 5 + len;
        if (hdr & 1) break;
    }
    if (raw.size() != static_cast<size_t>(h) * (1 + 3 * w)) fail("bad-image", path + ": truncated");
    Image img;
    img.width = w;
    img.height = h;
    img.px.resize(static_cast<size_t>(w) * h * 3);
    for (int y = 0; y < h; ++y)
        for (int i = 0; i < 3 * w; ++i) img.px[static_cast<size_t>(y) * w * 3 + i] = raw[y * (1 + 3 * w) + 1 + i] / 255.0;
    return img;
}

}  // namespace nexel
