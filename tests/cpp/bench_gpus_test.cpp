// run_benchmark_gpus (the B200 GPU-count axis of bench.hpp): G = 1, 2, 3 as
// contexts on the visible devices (device g mod count: on a one-GPU box every
// context shares device 0).  Checks the validation, the CSV layout (the
// reference's columns + alg_bytes, gb_per_s; blur and total rows), and that
// every frame's dense disparity + refocused image digest is identical for
// every G.  Prints the CSV.
#include <cstdio>
#include <string>
#include <vector>

#include "stereotk/bench.hpp"
#include "stereotk/pipeline.hpp"

using namespace stereotk;

#define CHECK(c)                                                  \
    do {                                                          \
        if (!(c)) {                                               \
            std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
            return 1;                                             \
        }                                                         \
    } while (0)

static RgbImage grey(int w, int h, unsigned seed, int shift) {
    RgbImage im(w, h);
    unsigned s = seed;
    std::vector<unsigned char> row(w + 64);
    for (int y = 0; y < h; ++y) {
        for (auto& v : row) v = (unsigned char)((s = s * 1103515245u + 12345u) >> 24);
        for (int x = 0; x < w; ++x) {
            const unsigned char v = (x / 9 + y / 7) % 3 == 0 ? row[x + shift] : (unsigned char)(40 * ((x / 13 + y / 11) % 5));
            im.at(x, y, 0) = im.at(x, y, 1) = im.at(x, y, 2) = v;
        }
    }
    return im;
}

int main() {
    std::vector<StereoPair> frames;
    for (int i = 0; i < 7; ++i) frames.push_back({grey(160, 96, 11 + i, 0), grey(160, 96, 11 + i, 3 + i % 4)});
    PipelineConfig cfg;
    cfg.k = 4;
    cfg.window = 9;
    cfg.max_disparity = 16;
    FocusSpec focus;
    focus.ranges = {{4, 9}};
    focus.sigma = 2.0;
    bool threw = false;
    try {
        run_benchmark_gpus(frames, {2, 3}, cfg, &focus);
    } catch (const ParamError&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        run_benchmark_gpus({}, {1}, cfg, &focus);
    } catch (const ParamError&) {
        threw = true;
    }
    CHECK(threw);
    const auto reports = run_benchmark_gpus(frames, {1, 2, 3}, cfg, &focus);
    CHECK(reports.size() == 3);
    for (const auto& r : reports) {
        CHECK(r.frames == 7);
        CHECK(r.digests.size() == 7);
        CHECK(r.digests == reports[0].digests);  // byte-identical outputs for every G
        CHECK(r.wall_ms > 0.0 && r.frames_per_s > 0.0);
        CHECK(r.times.match > 0.0 && r.blur > 0.0);
        CHECK(r.alg_bytes[0] == 8.0 * 160 * 96 * 7);
    }
    for (size_t i = 1; i < 7; ++i) CHECK(reports[0].digests[i] != reports[0].digests[0]);
    const std::string csv = benchmark_csv(reports);
    CHECK(csv.rfind("frames,gpus,stage,serial_ms,parallel_ms,speedup,alg_bytes,gb_per_s\n", 0) == 0);
    int lines = 0;
    for (char c : csv) lines += c == '\n';
    CHECK(lines == 1 + 8 * 3);  // header + 7 stages (blur included) + total per count
    CHECK(csv.find(",blur,") != std::string::npos && csv.find("7,3,total,") != std::string::npos);
    const auto pos = csv.find("7,1,total,");
    CHECK(pos != std::string::npos);
    const std::string row = csv.substr(pos, csv.find('\n', pos) - pos);
    // serial total compares against itself: speedup exactly 1
    CHECK(row.find(",1,") != std::string::npos);
    std::fputs(csv.c_str(), stdout);
    return 0;
}
