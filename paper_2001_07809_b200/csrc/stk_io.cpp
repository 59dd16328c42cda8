// stk_io.cpp -- frame and disparity file I/O for the drop-in (SURVEY.md §8f
// row 3): the reference's image_io.cpp / evaluate.cpp file entry points and
// tools/main.cpp's frame-pair discovery, as host code in libstk_b200.so.
//
//   load_image / load_gray / save_gray / save_rgb     image.hpp:55-79,
//                                                     image_io.cpp:14-241
//   save_disparity / load_disparity /
//   disparity_mask_path / load_ground_truth          evaluate.hpp:38-72,
//                                                     evaluate.cpp:76-90,136-229
//   list_frame_pairs / load_frames                    tools/main.cpp:247-284
//
// Binary PGM/PPM behave exactly as the reference (same accepted syntax, same
// exception class and message text); the CPU tests check that against the
// reference's own image_io.cpp compiled into oracle/_ref.  PNG: the reference
// links libpng's simplified API, which this image lacks, so PNG is decoded and
// encoded here directly over zlib (all colour types, bit depths 1-16, Adam7,
// tRNS; alpha is composited onto black in linear light and 16-bit / gAMA
// files are converted to 8-bit sRGB as libpng's simplified reader does).
// Frames go to the GPU through stk_frame_submit; decoding is host work.
#include <zlib.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <map>
#include <string>
#include <vector>

#include "stereotk/stereotk_b200.hpp"
#include "stk_b200.h"

namespace stk {
void set_thread_error(const std::string& msg);  // stk_capi.cu
}

namespace stereotk {
namespace {

namespace fs = std::filesystem;
using Bytes = std::vector<std::uint8_t>;

Bytes read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    Bytes b{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    if (in.bad()) throw IoError("read failed: " + path);
    return b;
}

void write_file(const std::string& path, const Bytes& b) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot open " + path + " for writing");
    out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
    if (!out) throw IoError("write failed: " + path);
}

// ------------------------------------------------------------------ PNM ----
// image_io.cpp:29-103: "P5"/"P6", then width, height, maxval as decimal
// fields, each optionally preceded by whitespace and '#' comment lines, then
// exactly one whitespace byte before the raster.
bool pnm_space(std::uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

struct Pnm {
    int channels = 0, width = 0, height = 0;
    std::size_t offset = 0;
};

Pnm pnm_header(const Bytes& b, const std::string& path, std::vector<std::string>* comments) {
    if (b.size() < 2 || b[0] != 'P' || (b[1] != '5' && b[1] != '6'))
        throw FormatError(path + ": not a binary PGM/PPM file");
    Pnm h;
    h.channels = b[1] == '6' ? 3 : 1;
    std::size_t p = 2;
    const std::size_t n = b.size();
    long v[3] = {0, 0, 0};
    for (long& f : v) {
        for (;;) {  // whitespace and comment lines before the field
            while (p < n && pnm_space(b[p])) ++p;
            if (p >= n || b[p] != '#') break;
            const std::size_t s = ++p;
            while (p < n && b[p] != '\n') ++p;
            if (comments) {
                std::size_t s2 = s;
                if (s2 < p && b[s2] == ' ') ++s2;
                comments->emplace_back(b.begin() + s2, b.begin() + p);
            }
        }
        if (p >= n || !std::isdigit(b[p])) throw FormatError(path + ": malformed PNM header");
        for (; p < n && std::isdigit(b[p]); ++p) {
            f = f * 10 + (b[p] - '0');
            if (f > (1L << 30)) throw FormatError(path + ": PNM header value out of range");
        }
    }
    if (p >= n || !pnm_space(b[p])) throw FormatError(path + ": malformed PNM header");
    h.offset = p + 1;
    if (v[0] <= 0 || v[1] <= 0) throw FormatError(path + ": bad PNM dimensions");
    if (v[2] <= 0 || v[2] > 255) throw FormatError(path + ": only 8-bit PNM rasters are supported");
    h.width = static_cast<int>(v[0]);
    h.height = static_cast<int>(v[1]);
    return h;
}

Bytes pnm_bytes(char magic, int w, int h, const std::vector<std::string>& comments,
                const std::uint8_t* data, std::size_t size) {
    std::string hdr = std::string("P") + magic + "\n";
    for (const std::string& c : comments) hdr += "# " + c + "\n";
    hdr += std::to_string(w) + " " + std::to_string(h) + "\n255\n";
    Bytes b(hdr.begin(), hdr.end());
    b.insert(b.end(), data, data + size);
    return b;
}

// ------------------------------------------------------------------ PNG ----
const std::uint8_t kPngSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};

bool is_png(const Bytes& b) { return b.size() >= 8 && std::memcmp(b.data(), kPngSig, 8) == 0; }

std::uint32_t be32(const std::uint8_t* p) {
    return (std::uint32_t(p[0]) << 24) | (std::uint32_t(p[1]) << 16) | (std::uint32_t(p[2]) << 8) | p[3];
}

void put32(Bytes& b, std::uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) b.push_back(static_cast<std::uint8_t>(v >> s));
}

// sRGB transfer curve (IEC 61966-2-1), used only when a file is not 8-bit
// sRGB-encoded (16-bit samples, a non-sRGB gAMA, or alpha composition).
double srgb_to_lin(double e) { return e <= 0.04045 ? e / 12.92 : std::pow((e + 0.055) / 1.055, 2.4); }
double lin_to_srgb(double l) {
    return l <= 0.0031308 ? 12.92 * l : 1.055 * std::pow(l, 1.0 / 2.4) - 0.055;
}
std::uint8_t q8(double e) {
    const long v = std::lround(e * 255.0);
    return static_cast<std::uint8_t>(std::clamp(v, 0L, 255L));
}

struct PngInfo {
    std::uint32_t w = 0, h = 0;
    int depth = 0, ctype = 0, interlace = 0;
    std::vector<std::uint8_t> plte;     // 3 * entries
    std::vector<std::uint8_t> trns;     // palette alphas, or the key sample(s)
    bool have_trns = false;
    int gamma = 0;                      // gAMA * 100000, 0 = absent
    bool srgb = false;
};

int png_channels(int ctype) {
    switch (ctype) {
        case 0: return 1;
        case 2: return 3;
        case 3: return 1;
        case 4: return 2;
        case 6: return 4;
    }
    return 0;
}

std::uint8_t paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return static_cast<std::uint8_t>(pa <= pb && pa <= pc ? a : (pb <= pc ? b : c));
}

// Reverse the per-row filters of one (sub)image in place; `raw` holds rows of
// 1 filter byte + stride bytes.
void unfilter(std::uint8_t* raw, std::size_t stride, std::uint32_t rows, int bpp, const std::string& path) {
    std::uint8_t* prev = nullptr;
    for (std::uint32_t y = 0; y < rows; ++y) {
        std::uint8_t* row = raw + y * (stride + 1);
        const int f = row[0];
        std::uint8_t* r = row + 1;
        switch (f) {
            case 0: break;
            case 1:
                for (std::size_t i = bpp; i < stride; ++i) r[i] += r[i - bpp];
                break;
            case 2:
                if (prev)
                    for (std::size_t i = 0; i < stride; ++i) r[i] += prev[i];
                break;
            case 3:
                for (std::size_t i = 0; i < stride; ++i) {
                    const int a = i >= std::size_t(bpp) ? r[i - bpp] : 0, b = prev ? prev[i] : 0;
                    r[i] += static_cast<std::uint8_t>((a + b) >> 1);
                }
                break;
            case 4:
                for (std::size_t i = 0; i < stride; ++i) {
                    const int a = i >= std::size_t(bpp) ? r[i - bpp] : 0, b = prev ? prev[i] : 0;
                    const int c = (prev && i >= std::size_t(bpp)) ? prev[i - bpp] : 0;
                    r[i] += paeth(a, b, c);
                }
                break;
            default: throw FormatError(path + ": bad PNG filter type " + std::to_string(f));
        }
        prev = r;
    }
}

// One sample of a row at pixel x, channel c, as a value in [0, 2^depth).
inline std::uint32_t sample(const std::uint8_t* r, std::uint32_t x, int c, int ch, int depth) {
    if (depth == 8) return r[x * ch + c];
    if (depth == 16) return (std::uint32_t(r[2 * (x * ch + c)]) << 8) | r[2 * (x * ch + c) + 1];
    const std::uint32_t bit = (x * ch + c) * depth;  // sub-byte depths have ch == 1
    return (r[bit >> 3] >> (8 - depth - (bit & 7))) & ((1u << depth) - 1);
}

RgbImage decode_png(const Bytes& b, const std::string& path) {
    PngInfo in;
    Bytes idat;
    std::size_t p = 8;
    bool got_ihdr = false, got_iend = false;
    while (!got_iend) {
        if (p + 12 > b.size()) throw FormatError(path + ": truncated PNG");
        const std::uint32_t len = be32(&b[p]);
        if (len > 0x7fffffffu || p + 12 + std::size_t(len) > b.size())
            throw FormatError(path + ": truncated PNG");
        const std::uint8_t* type = &b[p + 4];
        const std::uint8_t* d = &b[p + 8];
        const std::uint32_t crc = be32(d + len);
        if (static_cast<std::uint32_t>(crc32(crc32(0L, Z_NULL, 0), type, len + 4)) != crc)
            throw FormatError(path + ": PNG CRC error in chunk " + std::string(type, type + 4));
        const std::string t(type, type + 4);
        if (!got_ihdr && t != "IHDR") throw FormatError(path + ": PNG does not start with IHDR");
        if (t == "IHDR") {
            if (len != 13) throw FormatError(path + ": bad PNG IHDR");
            in.w = be32(d);
            in.h = be32(d + 4);
            in.depth = d[8];
            in.ctype = d[9];
            in.interlace = d[12];
            const int dp = in.depth, ct = in.ctype;
            const bool ok_depth = (ct == 0 && (dp == 1 || dp == 2 || dp == 4 || dp == 8 || dp == 16)) ||
                                  (ct == 3 && (dp == 1 || dp == 2 || dp == 4 || dp == 8)) ||
                                  ((ct == 2 || ct == 4 || ct == 6) && (dp == 8 || dp == 16));
            if (!ok_depth || d[10] != 0 || d[11] != 0 || in.interlace > 1)
                throw FormatError(path + ": unsupported PNG header (colour type " + std::to_string(ct) +
                                  ", depth " + std::to_string(dp) + ")");
            if (in.w == 0 || in.h == 0 || in.w > 0x7fffffffu || in.h > 0x7fffffffu ||
                std::uint64_t(in.w) * in.h > (std::uint64_t(1) << 32))
                throw FormatError(path + ": bad PNG dimensions");
            got_ihdr = true;
        } else if (t == "PLTE") {
            if (len % 3 || len == 0 || len > 768) throw FormatError(path + ": bad PNG palette");
            in.plte.assign(d, d + len);
        } else if (t == "tRNS") {
            in.trns.assign(d, d + len);
            in.have_trns = true;
        } else if (t == "gAMA") {
            if (len == 4) in.gamma = static_cast<int>(be32(d));
        } else if (t == "sRGB") {
            in.srgb = true;
        } else if (t == "IDAT") {
            idat.insert(idat.end(), d, d + len);
        } else if (t == "IEND") {
            got_iend = true;
        } else if (!(type[0] & 0x20)) {
            throw FormatError(path + ": unknown critical PNG chunk " + t);
        }
        p += 12 + std::size_t(len);
    }
    if (in.ctype == 3 && in.plte.empty()) throw FormatError(path + ": PNG palette missing");

    // Sub-images: the whole image, or the seven Adam7 passes.
    static const int a7[7][4] = {{0, 0, 8, 8}, {4, 0, 8, 8}, {0, 4, 4, 8}, {2, 0, 4, 4},
                                 {0, 2, 2, 4}, {1, 0, 2, 2}, {0, 1, 1, 2}};
    const int ch = png_channels(in.ctype);
    const int bits = ch * in.depth;
    const int bpp = std::max(1, bits / 8);
    struct Pass { std::uint32_t x0, y0, dx, dy, w, h; std::size_t stride, off; };
    std::vector<Pass> passes;
    std::size_t total = 0;
    for (int i = 0; i < (in.interlace ? 7 : 1); ++i) {
        Pass q{};
        if (in.interlace) {
            q = {std::uint32_t(a7[i][0]), std::uint32_t(a7[i][1]), std::uint32_t(a7[i][2]),
                 std::uint32_t(a7[i][3]), 0, 0, 0, 0};
        } else {
            q = {0, 0, 1, 1, 0, 0, 0, 0};
        }
        q.w = in.w > q.x0 ? (in.w - q.x0 + q.dx - 1) / q.dx : 0;
        q.h = in.h > q.y0 ? (in.h - q.y0 + q.dy - 1) / q.dy : 0;
        if (q.w == 0 || q.h == 0) continue;
        q.stride = (std::size_t(q.w) * bits + 7) / 8;
        q.off = total;
        total += (q.stride + 1) * q.h;
        passes.push_back(q);
    }
    Bytes raw(total);
    {
        z_stream zs{};
        if (inflateInit(&zs) != Z_OK) throw FormatError(path + ": zlib init failed");
        zs.next_in = idat.data();
        zs.avail_in = static_cast<uInt>(idat.size());
        zs.next_out = raw.data();
        zs.avail_out = static_cast<uInt>(raw.size());
        const int rc = inflate(&zs, Z_FINISH);
        const std::size_t got = raw.size() - zs.avail_out;
        inflateEnd(&zs);
        if ((rc != Z_STREAM_END && rc != Z_BUF_ERROR) || got != raw.size())
            throw FormatError(path + ": corrupt or truncated PNG image data");
    }

    // Per-sample conversion to 8-bit sRGB, as libpng's simplified reader:
    // 8-bit samples are taken as sRGB-encoded unless a gAMA chunk says
    // otherwise; 16-bit samples are linear unless gAMA / sRGB say otherwise.
    const int gamma = in.srgb ? 45455 : (in.gamma ? in.gamma : (in.depth == 16 ? 100000 : 45455));
    const bool srgb_like = std::abs(gamma - 45455) <= 45455 / 20;
    const std::uint32_t maxv = (1u << in.depth) - 1;
    auto to_lin = [&](std::uint32_t v) {  // sample -> linear light in [0, 1]
        const double e = double(v) / maxv;
        return srgb_like ? srgb_to_lin(e) : std::pow(e, 100000.0 / gamma);
    };
    // 8-bit (and expanded 1/2/4-bit) samples under a non-sRGB gAMA: libpng's
    // simplified reader corrects them to its sRGB output gamma (a 2.2 power)
    // with an 8-bit table, out = floor(255 (v/255)^(1/(2.2 g)) + 0.5) --
    // checked against libpng 1.6 (tests/golden/png_golden.npz); palette
    // entries go through the same table
    std::uint8_t gtab[256];
    for (int v = 0; v < 256; ++v)
        gtab[v] = srgb_like ? static_cast<std::uint8_t>(v)
                            : static_cast<std::uint8_t>(std::floor(
                                  255.0 * std::pow(v / 255.0, 100000.0 / (2.2 * gamma)) + 0.5));
    auto to8 = [&](std::uint32_t v) -> std::uint8_t {
        if (in.depth == 8) return gtab[v];
        if (in.depth < 8) return gtab[v * 255 / maxv];
        if (srgb_like) return static_cast<std::uint8_t>((v * 255 + 32895) >> 16);  // 16-bit sRGB
        return q8(lin_to_srgb(to_lin(v)));
    };
    auto composite = [&](std::uint32_t v, double alpha) -> std::uint8_t {  // onto black
        return q8(lin_to_srgb(to_lin(v) * alpha));
    };

    RgbImage img(static_cast<int>(in.w), static_cast<int>(in.h));
    const std::uint32_t amax = in.depth == 16 ? 65535 : 255;
    for (const Pass& q : passes) {
        std::uint8_t* base = raw.data() + q.off;
        unfilter(base, q.stride, q.h, bpp, path);
        for (std::uint32_t yy = 0; yy < q.h; ++yy) {
            const std::uint8_t* r = base + yy * (q.stride + 1) + 1;
            const std::uint32_t y = q.y0 + yy * q.dy;
            for (std::uint32_t xx = 0; xx < q.w; ++xx) {
                const std::uint32_t x = q.x0 + xx * q.dx;
                std::uint8_t* o = &img.data[(std::size_t(y) * in.w + x) * 3];
                if (in.ctype == 3) {
                    const std::uint32_t i = sample(r, xx, 0, 1, in.depth);
                    if (3 * i + 2 >= in.plte.size()) throw FormatError(path + ": PNG palette index out of range");
                    const std::uint8_t* c = &in.plte[3 * i];
                    const int a = i < in.trns.size() ? in.trns[i] : 255;
                    for (int k = 0; k < 3; ++k) o[k] = a == 255 ? gtab[c[k]] : q8(lin_to_srgb(srgb_to_lin(c[k] / 255.0) * a / 255.0));
                    continue;
                }
                std::uint32_t s[4] = {0, 0, 0, amax};
                for (int c = 0; c < ch; ++c) s[c] = sample(r, xx, c, ch, in.depth);
                std::uint32_t g[3];
                if (ch <= 2) {
                    g[0] = g[1] = g[2] = s[0];
                } else {
                    g[0] = s[0]; g[1] = s[1]; g[2] = s[2];
                }
                std::uint32_t alpha = ch == 2 ? s[1] : (ch == 4 ? s[3] : amax);
                if (in.have_trns && in.ctype == 0 && in.trns.size() >= 2 && s[0] == ((in.trns[0] << 8) | in.trns[1]))
                    alpha = 0;
                if (in.have_trns && in.ctype == 2 && in.trns.size() >= 6 &&
                    s[0] == ((in.trns[0] << 8) | in.trns[1]) && s[1] == ((in.trns[2] << 8) | in.trns[3]) &&
                    s[2] == ((in.trns[4] << 8) | in.trns[5]))
                    alpha = 0;
                for (int k = 0; k < 3; ++k)
                    o[k] = alpha == amax ? to8(g[k]) : composite(g[k], double(alpha) / amax);
            }
        }
    }
    return img;
}

// 8-bit RGB, non-interlaced; per row the filter with the smallest sum of
// |signed residuals| (the usual heuristic); one IDAT.
Bytes encode_png(const RgbImage& img) {
    const std::size_t stride = std::size_t(img.width) * 3;
    Bytes filt((stride + 1) * img.height);
    std::vector<std::uint8_t> cand[5];
    for (auto& c : cand) c.resize(stride);
    for (int y = 0; y < img.height; ++y) {
        const std::uint8_t* r = &img.data[y * stride];
        const std::uint8_t* pr = y ? &img.data[(y - 1) * stride] : nullptr;
        long best = -1;
        int bf = 0;
        for (int f = 0; f < 5; ++f) {
            long cost = 0;
            for (std::size_t i = 0; i < stride; ++i) {
                const int a = i >= 3 ? r[i - 3] : 0, b = pr ? pr[i] : 0, c = (pr && i >= 3) ? pr[i - 3] : 0;
                int pred = 0;
                switch (f) {
                    case 1: pred = a; break;
                    case 2: pred = b; break;
                    case 3: pred = (a + b) >> 1; break;
                    case 4: pred = paeth(a, b, c); break;
                }
                const std::uint8_t v = static_cast<std::uint8_t>(r[i] - pred);
                cand[f][i] = v;
                cost += v < 128 ? v : 256 - v;
            }
            if (best < 0 || cost < best) {
                best = cost;
                bf = f;
            }
        }
        filt[y * (stride + 1)] = static_cast<std::uint8_t>(bf);
        std::memcpy(&filt[y * (stride + 1) + 1], cand[bf].data(), stride);
    }
    uLongf zlen = compressBound(static_cast<uLong>(filt.size()));
    Bytes z(zlen);
    if (compress2(z.data(), &zlen, filt.data(), static_cast<uLong>(filt.size()), Z_DEFAULT_COMPRESSION) != Z_OK)
        throw IoError("png: deflate failed");
    z.resize(zlen);

    Bytes out(kPngSig, kPngSig + 8);
    auto chunk = [&](const char* type, const std::uint8_t* d, std::size_t n) {
        put32(out, static_cast<std::uint32_t>(n));
        const std::size_t s = out.size();
        out.insert(out.end(), type, type + 4);
        out.insert(out.end(), d, d + n);
        put32(out, static_cast<std::uint32_t>(crc32(crc32(0L, Z_NULL, 0), &out[s], static_cast<uInt>(n + 4))));
    };
    Bytes ihdr;
    put32(ihdr, static_cast<std::uint32_t>(img.width));
    put32(ihdr, static_cast<std::uint32_t>(img.height));
    ihdr.insert(ihdr.end(), {8, 2, 0, 0, 0});
    chunk("IHDR", ihdr.data(), ihdr.size());
    const std::uint8_t intent = 0;
    chunk("sRGB", &intent, 1);
    chunk("IDAT", z.data(), z.size());
    chunk("IEND", nullptr, 0);
    return out;
}

std::string lower_ext(const std::string& path) {
    const std::size_t dot = path.find_last_of('.');
    if (dot == std::string::npos) return "";
    std::string e = path.substr(dot);
    for (char& c : e) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return e;
}

// std::to_string(scale) with trailing zeros (and a bare '.') trimmed, as
// evaluate.cpp:162-171 prints the scale comment.
std::string scale_text(double s) {
    std::string t = std::to_string(s);
    if (t.find('.') == std::string::npos) return t;
    while (!t.empty() && t.back() == '0') t.pop_back();
    if (!t.empty() && t.back() == '.') t.pop_back();
    return t;
}

}  // namespace

// ------------------------------------------------------------ image.hpp ----
RgbImage load_image(const std::string& path) {
    const Bytes b = read_file(path);
    if (is_png(b)) return decode_png(b, path);
    const Pnm h = pnm_header(b, path, nullptr);
    const std::size_t n = std::size_t(h.width) * h.height * h.channels;
    if (b.size() - h.offset < n) throw FormatError(path + ": truncated PNM raster");
    RgbImage img(h.width, h.height);
    const std::uint8_t* src = b.data() + h.offset;
    if (h.channels == 3) {
        std::memcpy(img.data.data(), src, n);
    } else {
        for (std::size_t i = 0; i < n; ++i) img.data[3 * i] = img.data[3 * i + 1] = img.data[3 * i + 2] = src[i];
    }
    return img;
}

GrayImage load_gray(const std::string& path, std::vector<std::string>* comments) {
    const Bytes b = read_file(path);
    if (is_png(b)) {
        const RgbImage rgb = decode_png(b, path);
        GrayImage g(rgb.width, rgb.height);
        for (std::size_t i = 0; i < g.data.size(); ++i) {
            const std::uint8_t* p = &rgb.data[3 * i];
            if (p[0] != p[1] || p[0] != p[2])
                throw FormatError(path + ": PNG has colour pixels, expected a single-channel image");
            g.data[i] = p[0];
        }
        return g;
    }
    const Pnm h = pnm_header(b, path, comments);
    if (h.channels != 1) throw FormatError(path + ": expected a single-channel (P5) file");
    const std::size_t n = std::size_t(h.width) * h.height;
    if (b.size() - h.offset < n) throw FormatError(path + ": truncated PGM raster");
    GrayImage g(h.width, h.height);
    std::memcpy(g.data.data(), b.data() + h.offset, n);
    return g;
}

void save_gray(const GrayImage& image, const std::string& path, const std::vector<std::string>& comments) {
    write_file(path, pnm_bytes('5', image.width, image.height, comments, image.data.data(), image.data.size()));
}

void save_rgb(const RgbImage& image, const std::string& path) {
    if (lower_ext(path) == ".png") {
        Bytes png;
        try {
            png = encode_png(image);
        } catch (const IoError& e) {
            throw IoError(path + ": " + e.what());
        }
        write_file(path, png);
        return;
    }
    write_file(path, pnm_bytes('6', image.width, image.height, {}, image.data.data(), image.data.size()));
}

// --------------------------------------------------------- evaluate.hpp ----
DisparityMap load_ground_truth(const std::string& path, double scale) {
    if (!(scale > 0.0))
        throw ParamError("load_ground_truth: scale must be positive, got " + std::to_string(scale));
    const GrayImage raw = load_gray(path);
    DisparityMap t(raw.width, raw.height);
    for (std::size_t i = 0; i < raw.data.size(); ++i)
        if (raw.data[i]) t.values[i] = static_cast<std::int16_t>(std::lround(raw.data[i] / scale));
    return t;
}

std::string disparity_mask_path(const std::string& path) {
    const std::size_t slash = path.find_last_of("/\\");
    const std::size_t dot = path.find_last_of('.');
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return path + ".mask.pgm";
    return path.substr(0, dot) + ".mask" + path.substr(dot);
}

void save_disparity(const DisparityMap& map, const std::string& path, double output_scale) {
    if (!(output_scale > 0.0))
        throw ParamError("save_disparity: scale must be positive, got " + std::to_string(output_scale));
    GrayImage vals(map.width, map.height), known(map.width, map.height);
    for (std::size_t i = 0; i < map.values.size(); ++i) {
        const std::int16_t d = map.values[i];
        if (d < 0) continue;
        const long s = std::lround(d * output_scale);
        if (s < 0 || s > 255)
            throw ParamError("save_disparity: disparity " + std::to_string(d) + " at scale " +
                             std::to_string(output_scale) + " does not fit in 8 bits");
        vals.data[i] = static_cast<std::uint8_t>(s);
        known.data[i] = 255;
    }
    save_gray(vals, path, {"scale " + scale_text(output_scale)});
    save_gray(known, disparity_mask_path(path));
}

DisparityMap load_disparity(const std::string& path, double fallback_scale) {
    std::vector<std::string> comments;
    const GrayImage raw = load_gray(path, &comments);
    double scale = fallback_scale > 0.0 ? fallback_scale : 1.0;
    for (const std::string& c : comments) {
        if (c.rfind("scale ", 0) != 0) continue;
        try {
            scale = std::stod(c.substr(6));
        } catch (const std::exception&) {
            throw FormatError(path + ": bad scale comment '" + c + "'");
        }
        if (!(scale > 0.0)) throw FormatError(path + ": non-positive scale comment");
        break;
    }
    const std::string mpath = disparity_mask_path(path);
    DisparityMap m(raw.width, raw.height);
    const bool have_mask = fs::exists(mpath);
    GrayImage known;
    if (have_mask) {
        known = load_gray(mpath);
        if (known.width != raw.width || known.height != raw.height)
            throw FormatError(mpath + ": mask size does not match " + path);
    }
    for (std::size_t i = 0; i < raw.data.size(); ++i)
        if (have_mask ? known.data[i] != 0 : raw.data[i] != 0)
            m.values[i] = static_cast<std::int16_t>(std::lround(raw.data[i] / scale));
    return m;
}

// -------------------------------------------- frame pairs (main.cpp:247-284) --
std::vector<std::pair<std::string, std::string>> list_frame_pairs(const std::string& dir) {
    if (!fs::is_directory(dir)) throw IoError("not a directory: " + dir);
    static const char* kExt[] = {".png", ".ppm", ".pgm"};
    std::vector<fs::path> names;
    for (const fs::directory_entry& e : fs::directory_iterator(dir))
        if (e.is_regular_file()) names.push_back(e.path());
    std::sort(names.begin(), names.end());  // deterministic when a stem has several extensions
    std::map<std::string, std::pair<std::string, std::string>> found;
    for (const fs::path& p : names) {
        const std::string name = p.filename().string();
        for (const char* ext : kExt) {
            const std::string suf = std::string("_L") + ext;
            if (name.size() <= suf.size() || name.compare(name.size() - suf.size(), suf.size(), suf) != 0)
                continue;
            const std::string stem = name.substr(0, name.size() - suf.size());
            const fs::path right = p.parent_path() / (stem + "_R" + ext);
            if (fs::exists(right)) found[stem] = {p.string(), right.string()};
        }
    }
    if (found.empty()) throw ParamError("no *_L/_R frame pairs found in " + dir);
    std::vector<std::pair<std::string, std::string>> out;
    for (const auto& kv : found) out.push_back(kv.second);
    return out;
}

std::vector<StereoPair> load_frames(const std::string& dir) {
    std::vector<StereoPair> frames;
    for (const auto& lr : list_frame_pairs(dir)) frames.push_back({load_image(lr.first), load_image(lr.second)});
    return frames;
}

}  // namespace stereotk

// ================================================================ C-ABI ====
using stereotk::Bytes;
using stereotk::be32;
using stereotk::is_png;
using stereotk::png_channels;

namespace {

template <class F>
stk_status guard(F&& f) {
    try {
        f();
        return STK_OK;
    } catch (const stereotk::ParamError& e) {
        stk::set_thread_error(e.what());
        return STK_EPARAM;
    } catch (const stereotk::IoError& e) {
        stk::set_thread_error(e.what());
        return STK_EIO;
    } catch (const stereotk::FormatError& e) {
        stk::set_thread_error(e.what());
        return STK_EFORMAT;
    } catch (const std::bad_alloc&) {
        stk::set_thread_error("out of host memory");
        return STK_EINTERNAL;
    } catch (const std::exception& e) {
        stk::set_thread_error(e.what());
        return STK_EINTERNAL;
    }
}

void copy_str(const std::string& s, char* out, size_t cap, size_t* need) {
    if (need) *need = s.size() + 1;
    if (out && cap) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
}

std::vector<std::string> split_lines(const char* s) {
    std::vector<std::string> v;
    if (!s) return v;
    std::string cur;
    for (; *s; ++s) {
        if (*s == '\n') {
            v.push_back(cur);
            cur.clear();
        } else {
            cur += *s;
        }
    }
    if (!cur.empty()) v.push_back(cur);
    return v;
}

void check_dims(const char* what, int w, int h, int gw, int gh) {
    if (w != gw || h != gh)
        throw stereotk::ParamError(std::string(what) + ": buffer is " + std::to_string(w) + "x" +
                                   std::to_string(h) + ", file is " + std::to_string(gw) + "x" +
                                   std::to_string(gh));
}

}  // namespace

extern "C" {

stk_status stk_image_probe(const char* path, int* w, int* h, int* channels) {
    return guard([&] {
        if (!path) throw stereotk::ParamError("stk_image_probe: null path");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw stereotk::IoError(std::string("cannot open ") + path);
        Bytes b(64);
        in.read(reinterpret_cast<char*>(b.data()), 64);
        b.resize(static_cast<size_t>(in.gcount()));
        int W = 0, H = 0, C = 0;
        if (is_png(b)) {
            // the IHDR must be intact (length, type, CRC) before its sizes are trusted
            if (b.size() < 33 || be32(&b[8]) != 13 || std::memcmp(&b[12], "IHDR", 4) != 0 ||
                static_cast<std::uint32_t>(crc32(crc32(0L, Z_NULL, 0), &b[12], 17)) != be32(&b[29]))
                throw stereotk::FormatError(std::string(path) + ": truncated or corrupt PNG header");
            const std::uint32_t pw = be32(&b[16]), ph = be32(&b[20]);
            if (pw == 0 || ph == 0 || pw > 0x7fffffffu || ph > 0x7fffffffu ||
                std::uint64_t(pw) * ph > (std::uint64_t(1) << 32))
                throw stereotk::FormatError(std::string(path) + ": bad PNG dimensions");
            W = static_cast<int>(pw);
            H = static_cast<int>(ph);
            C = png_channels(b[25]) >= 3 || b[25] == 3 ? 3 : 1;
        } else {
            // the header from the first MiB (the whole file if the header --
            // which may carry long comment lines -- does not fit)
            Bytes head(1 << 20);
            in.clear();
            in.seekg(0);
            in.read(reinterpret_cast<char*>(head.data()), static_cast<std::streamsize>(head.size()));
            head.resize(static_cast<size_t>(in.gcount()));
            stereotk::Pnm hd;
            try {
                hd = stereotk::pnm_header(head, path, nullptr);
            } catch (const stereotk::FormatError&) {
                if (head.size() < (1u << 20)) throw;
                hd = stereotk::pnm_header(stereotk::read_file(path), path, nullptr);
            }
            W = hd.width;
            H = hd.height;
            C = hd.channels;
        }
        if (w) *w = W;
        if (h) *h = H;
        if (channels) *channels = C;
    });
}

stk_status stk_load_image(const char* path, uint8_t* rgb, int w, int h) {
    return guard([&] {
        const stereotk::RgbImage img = stereotk::load_image(path);
        check_dims("stk_load_image", w, h, img.width, img.height);
        std::memcpy(rgb, img.data.data(), img.data.size());
    });
}

stk_status stk_load_gray(const char* path, uint8_t* gray, int w, int h, char* comments, size_t cap,
                         size_t* need) {
    return guard([&] {
        std::vector<std::string> c;
        const stereotk::GrayImage img = stereotk::load_gray(path, &c);
        check_dims("stk_load_gray", w, h, img.width, img.height);
        std::memcpy(gray, img.data.data(), img.data.size());
        std::string joined;
        for (const auto& s : c) joined += s + "\n";
        copy_str(joined, comments, cap, need);
    });
}

stk_status stk_save_gray(const char* path, const uint8_t* gray, int w, int h, const char* comments) {
    return guard([&] {
        stereotk::GrayImage img(w, h);
        std::memcpy(img.data.data(), gray, img.data.size());
        stereotk::save_gray(img, path, split_lines(comments));
    });
}

stk_status stk_save_rgb(const char* path, const uint8_t* rgb, int w, int h) {
    return guard([&] {
        stereotk::RgbImage img(w, h);
        std::memcpy(img.data.data(), rgb, img.data.size());
        stereotk::save_rgb(img, path);
    });
}

stk_status stk_save_disparity(const char* path, const int16_t* d, int w, int h, double scale) {
    return guard([&] {
        stereotk::DisparityMap m(w, h);
        std::memcpy(m.values.data(), d, m.values.size() * 2);
        stereotk::save_disparity(m, path, scale);
    });
}

stk_status stk_load_disparity(const char* path, int16_t* d, int w, int h, double fallback_scale) {
    return guard([&] {
        const stereotk::DisparityMap m = stereotk::load_disparity(path, fallback_scale);
        check_dims("stk_load_disparity", w, h, m.width, m.height);
        std::memcpy(d, m.values.data(), m.values.size() * 2);
    });
}

stk_status stk_load_ground_truth(const char* path, int16_t* d, int w, int h, double scale) {
    return guard([&] {
        const stereotk::DisparityMap m = stereotk::load_ground_truth(path, scale);
        check_dims("stk_load_ground_truth", w, h, m.width, m.height);
        std::memcpy(d, m.values.data(), m.values.size() * 2);
    });
}

stk_status stk_disparity_mask_path(const char* path, char* out, size_t cap, size_t* need) {
    return guard([&] { copy_str(stereotk::disparity_mask_path(path), out, cap, need); });
}

stk_status stk_list_frame_pairs(const char* dir, char* out, size_t cap, size_t* need, int* count) {
    return guard([&] {
        const auto pairs = stereotk::list_frame_pairs(dir);
        std::string s;
        for (const auto& lr : pairs) s += lr.first + "\t" + lr.second + "\n";
        copy_str(s, out, cap, need);
        if (count) *count = static_cast<int>(pairs.size());
    });
}

}  // extern "C"
