// Drop-in check: code written against the reference's stereotk:: headers
// compiles unchanged against include/stereotk/ and runs on the B200 through
// libstk_b200.so.  The checks restate reference tests (file:line cited);
// the last step dumps one refocused frame so the pytest driver can compare
// it byte for byte with the C-ABI / golden path.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "stereotk/boundary.hpp"
#include "stereotk/error.hpp"
#include "stereotk/pipeline.hpp"
#include "stereotk/refocus.hpp"
#include "stereotk/segmentation.hpp"
#include "stereotk/stereo.hpp"

using namespace stereotk;

static int failures = 0;
#define CHECK(c)                                                       \
    do {                                                               \
        if (!(c)) {                                                    \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                \
        }                                                              \
    } while (0)

// synthetic.cpp:90-104 restated (raw mt19937 draws)
static StereoPair rectangle_scene_pair(int width, int height, int shift, std::uint32_t seed) {
    std::mt19937 rng(seed);
    RgbImage wide(width + shift, height);
    auto rect = [&](int x0, int y0, int x1, int y1, int base, int spread) {
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                const auto v = static_cast<std::uint8_t>(base + static_cast<int>(rng() % spread));
                wide.at(x, y, 0) = wide.at(x, y, 1) = wide.at(x, y, 2) = v;
            }
    };
    rect(0, 0, wide.width, height, 20, 50);
    rect(width * 2 / 10, height * 2 / 10, width * 4 / 10, height * 5 / 10, 150, 70);
    rect(width * 6 / 10, height * 55 / 100, width * 9 / 10, height * 85 / 100, 150, 70);
    StereoPair p{RgbImage(width, height), RgbImage(width, height)};
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x)
            for (int c = 0; c < 3; ++c) {
                p.left.at(x, y, c) = wide.at(x, y, c);
                p.right.at(x, y, c) = wide.at(x + shift, y, c);
            }
    return p;
}

int main(int argc, char** argv) {
    // mismatched frames (test_pipeline.cpp:12-24)
    try {
        run_depth_pipeline(RgbImage(64, 48), RgbImage(32, 48), PipelineConfig{});
        CHECK(false);
    } catch (const ParamError& e) {
        const std::string m = e.what();
        CHECK(m.find("64x48") != std::string::npos && m.find("32x48") != std::string::npos);
    }
    // configuration limits (test_pipeline.cpp:26-46)
    PipelineConfig bad;
    bad.window = 4;
    bool threw = false;
    try {
        validate_config(bad);
    } catch (const ParamError&) {
        threw = true;
    }
    CHECK(threw);
    // two bins -> two clusters (test_segmentation.cpp:43-57)
    GrayImage two(5, 2);
    two.data = {10, 10, 10, 10, 10, 200, 200, 200, 200, 200};
    Clustering cl = kmeans_histogram(build_histogram(two), 2);
    CHECK(cl.k() == 2 && cl.centers[0] == 10.0 && cl.centers[1] == 200.0);
    // prune {1, 2, 97} at 4 % (test_boundary.cpp:204-235)
    BoundaryMask m(24, 16);
    for (int y = 0; y <= 9; ++y)
        for (int x = 0; x <= 9; ++x) m.at(x, y) = 1;
    m.at(9, 9) = m.at(8, 9) = m.at(9, 8) = 0;
    m.at(15, 14) = 1;
    m.at(20, 3) = m.at(21, 3) = 1;
    CHECK(prune_components(m, 0.04).count() == 97);
    ComponentTable t = label_components(m);
    CHECK(t.sizes.size() == 3 && t.by_size.size() == 3 && t.sizes[t.by_size[2]] == 97);
    // translation recovery (acceptance_main.cpp:443-489)
    for (int s = 1; s <= 8; ++s) {
        StereoPair p = rectangle_scene_pair(160, 120, s, 700 + s);
        PipelineConfig cfg;
        cfg.k = 2;
        cfg.window = 9;
        cfg.max_disparity = 16;
        StageTimes times;
        DepthResult d = run_depth_pipeline(p.left, p.right, cfg, &times);
        CHECK(times.total() > 0.0);
        CHECK(d.stats.matched > 0);
        CHECK(d.dense.known_count() >= d.sparse.known_count());
        CHECK(d.clustering.k() == 2 && d.labels.width == 160);
    }
    // refocus keeps focused pixels (test_pipeline.cpp:140-168)
    StereoPair p = rectangle_scene_pair(96, 72, 4, 64);
    PipelineConfig cfg;
    cfg.k = 2;
    cfg.max_disparity = 8;
    FocusSpec focus;
    focus.ranges = {{4, 4}};
    DepthResult depth;
    RgbImage out = run_refocus_pipeline(p.left, p.right, cfg, focus, 0, &depth);
    int sharp = 0;
    for (int y = 0; y < 72; ++y)
        for (int x = 0; x < 96; ++x)
            if (depth.dense.known(x, y) && depth.dense.at(x, y) == 4) {
                ++sharp;
                for (int c = 0; c < 3; ++c) CHECK(out.at(x, y, c) == p.left.at(x, y, c));
            }
    CHECK(sharp > 0);
    // non-Gaussian weights take the exact 2-D path; a Gaussian equals it within 1 LSB
    GaussianKernel box;
    box.size = 3;
    box.weights.assign(9, 1.0 / 9.0);
    GrayImage all(96, 72);
    for (auto& v : all.data) v = 1;
    RgbImage b = selective_blur(p.left, all, box);
    CHECK(b.width == 96);
    {  // evaluate.hpp (test_evaluate.cpp:38-50, 125-143, 205-227)
        DisparityMap c(2, 2), t(2, 2);
        c.values = {5, 5, 7, 2};
        t.values = {5, 6, 9, 2};
        EvalResult r = bad_pixel_rate(c, t, 1.0);
        CHECK(r.bad_pixel_rate == 0.25 && r.compared == 4 && r.excluded == 0 && r.delta_d == 1.0);
        CHECK(bad_pixel_rate(c, t, 0.0).bad_pixel_rate == 0.5);
        bool threw = false;
        try {
            bad_pixel_rate(c, DisparityMap(2, 3), 1.0);
        } catch (const ParamError&) {
            threw = true;
        }
        CHECK(threw);
        EvalResult e;
        e.bad_pixel_rate = 0.25;
        e.compared = 4;
        e.excluded = 0;
        e.delta_d = 1.0;
        CHECK(eval_report_json(e) == "{\"bad_pixel_rate\":0.25,\"compared\":4,\"delta_d\":1.0,\"excluded\":0}");
        StereoPair tn = rectangle_scene_pair(24, 20, 3, 55);
        GrayImage gl = rgb_to_lightness(tn.left), gr = rgb_to_lightness(tn.right);
        MatchConfig mc;
        mc.window = 3;
        mc.max_disparity = 6;
        BoundaryMask every(24, 20);
        for (auto& v : every.mask) v = 1;
        CHECK(dense_sad_baseline(gl, gr, mc).values == match_boundary_pixels(gl, gr, every, mc).values);
    }
    {  // bench.hpp (test_parallel.cpp:78-117): validation and the CSV layout
        std::vector<StereoPair> frames;
        PipelineConfig bc;
        bc.max_disparity = 8;
        auto throws = [&](const std::vector<int>& wc) {
            try {
                run_benchmark(frames, wc, bc);
            } catch (const ParamError&) {
                return true;
            }
            return false;
        };
        CHECK(throws({1}));  // no frames
        frames.push_back(rectangle_scene_pair(96, 72, 4, 4));
        CHECK(throws({}));
        CHECK(throws({2, 4}));
        CHECK(throws({1, 0}));
        auto reports = run_benchmark(frames, {1, 2}, bc);
        const std::string csv = benchmark_csv(reports);
        CHECK(csv.rfind("frames,workers,stage,serial_ms,parallel_ms,speedup\n", 0) == 0);
        int lines = 0;
        for (char ch : csv) lines += ch == '\n';
        CHECK(lines == 1 + 7 * 2);
        CHECK(csv.find(",total,") != std::string::npos && csv.find(",match,") != std::string::npos);
        const auto pos = csv.find("1,1,total,");
        CHECK(pos != std::string::npos);
        const std::string row = csv.substr(pos, csv.find('\n', pos) - pos);
        CHECK(row.substr(row.rfind(',') + 1) == "1");
        CHECK(reports[0].times.match > 0.0 && reports[1].speedup > 0.0);
    }
    if (argc > 1) {  // dump the rect(96,72,4,63) frame for the byte comparison
        StereoPair q = rectangle_scene_pair(96, 72, 4, 63);
        PipelineConfig c2;
        c2.k = 2;
        c2.max_disparity = 8;
        FocusSpec f2;
        f2.ranges = {{3, 8}};
        DepthResult d2;
        RgbImage o2 = run_refocus_pipeline(q.left, q.right, c2, f2, 0, &d2);
        FILE* fp = std::fopen(argv[1], "wb");
        std::fwrite(d2.dense.values.data(), 2, d2.dense.values.size(), fp);
        std::fwrite(o2.data.data(), 1, o2.data.size(), fp);
        std::fwrite(b.data.data(), 1, b.data.size(), fp);
        std::fclose(fp);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
