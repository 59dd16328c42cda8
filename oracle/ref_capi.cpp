// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" adapter over the UNMODIFIED reference library, compiled
// from the reference's own sources where they lie under /root/reference/proj
// (see oracle/Makefile; output goes to oracle/_ref/, which is git-ignored).
// Python tests and bench.py's reference arm load it through ctypes to obtain
// the reference's exact outputs and timings.  Nothing here is product code.
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "stereotk/boundary.hpp"
#include "stereotk/error.hpp"
#include "stereotk/evaluate.hpp"
#include "stereotk/image.hpp"
#include "stereotk/parallel.hpp"
#include "stereotk/pipeline.hpp"
#include "stereotk/reconstruct.hpp"
#include "stereotk/refocus.hpp"
#include "stereotk/segmentation.hpp"
#include "stereotk/stereo.hpp"
#include "synthetic.hpp"

using namespace stereotk;

namespace {
thread_local std::string g_err;

RgbImage rgb_in(const uint8_t* p, int w, int h) {
    RgbImage im(w, h);
    std::memcpy(im.data.data(), p, im.data.size());
    return im;
}
GrayImage gray_in(const uint8_t* p, int w, int h) {
    GrayImage im(w, h);
    std::memcpy(im.data.data(), p, im.data.size());
    return im;
}
BoundaryMask mask_in(const uint8_t* p, int w, int h) {
    BoundaryMask m(w, h);
    std::memcpy(m.mask.data(), p, m.mask.size());
    return m;
}
DisparityMap disp_in(const int16_t* p, int w, int h) {
    DisparityMap d(w, h);
    std::memcpy(d.values.data(), p, d.values.size() * 2);
    return d;
}

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ParamError& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
}  // namespace

// image_io.cpp is compiled from the reference sources against
// oracle/pngstub/png.h (libpng is absent): its PGM/PPM code runs unmodified,
// PNG entries throw.  File entry points report the exception class:
// 0 ok, -1 ParamError, -3 IoError, -4 FormatError, -2 anything else.
namespace {
const void* im_data(const RgbImage& i) { return i.data.data(); }
const void* im_data(const GrayImage& i) { return i.data.data(); }
const void* im_data(const DisparityMap& i) { return i.values.data(); }

template <typename Fn>
int io_guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ParamError& e) {
        g_err = e.what();
        return -1;
    } catch (const IoError& e) {
        g_err = e.what();
        return -3;
    } catch (const FormatError& e) {
        g_err = e.what();
        return -4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
// Two-call pattern: buf == nullptr -> only *w/*h are reported.
template <typename Img>
void copy_out(const Img& im, int* w, int* h, void* buf, std::size_t elem_bytes) {
    *w = im.width;
    *h = im.height;
    if (buf) std::memcpy(buf, im_data(im), static_cast<std::size_t>(im.width) * im.height * elem_bytes);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_load_image(const char* path, int* w, int* h, uint8_t* rgb) {
    return io_guard([&] { copy_out(load_image(path), w, h, rgb, 3); });
}
int ref_load_gray(const char* path, int* w, int* h, uint8_t* gray, char* comments, int cap) {
    return io_guard([&] {
        std::vector<std::string> c;
        copy_out(load_gray(path, &c), w, h, gray, 1);
        std::string j;
        for (const auto& s : c) j += s + "\n";
        if (comments && cap > 0) std::snprintf(comments, cap, "%s", j.c_str());
    });
}
int ref_save_gray(const char* path, const uint8_t* gray, int w, int h, const char* comment) {
    return io_guard([&] {
        std::vector<std::string> c;
        if (comment && *comment) c.push_back(comment);
        save_gray(gray_in(gray, w, h), path, c);
    });
}
int ref_save_rgb(const char* path, const uint8_t* rgb, int w, int h) {
    return io_guard([&] { save_rgb(rgb_in(rgb, w, h), path); });
}
int ref_save_disparity(const char* path, const int16_t* d, int w, int h, double scale) {
    return io_guard([&] { save_disparity(disp_in(d, w, h), path, scale); });
}
int ref_load_disparity(const char* path, double fallback, int* w, int* h, int16_t* d) {
    return io_guard([&] { copy_out(load_disparity(path, fallback), w, h, d, 2); });
}
int ref_load_ground_truth(const char* path, double scale, int* w, int* h, int16_t* d) {
    return io_guard([&] { copy_out(load_ground_truth(path, scale), w, h, d, 2); });
}

int ref_dense_sad_baseline(const uint8_t* l, const uint8_t* r, int w, int h, int window, int max_d,
                           int workers, int16_t* out) {
    return guard([&] {
        MatchConfig c;
        c.window = window;
        c.max_disparity = max_d;
        const DisparityMap m = dense_sad_baseline(gray_in(l, w, h), gray_in(r, w, h), c, workers);
        std::memcpy(out, m.values.data(), m.values.size() * 2);
    });
}

int ref_bad_pixel_rate(const int16_t* comp, const int16_t* truth, int w, int h, double delta,
                       int workers, double* rate, uint64_t* compared, uint64_t* excluded,
                       char* json, int json_cap) {
    return guard([&] {
        const EvalResult e = bad_pixel_rate(disp_in(comp, w, h), disp_in(truth, w, h), delta, workers);
        *rate = e.bad_pixel_rate;
        *compared = e.compared;
        *excluded = e.excluded;
        const std::string js = eval_report_json(e);
        std::snprintf(json, json_cap, "%s", js.c_str());
    });
}

int ref_lightness(const uint8_t* rgb, int w, int h, int workers, uint8_t* gray) {
    return guard([&] {
        GrayImage g = rgb_to_lightness(rgb_in(rgb, w, h), workers);
        std::memcpy(gray, g.data.data(), g.data.size());
    });
}

int ref_histogram(const uint8_t* gray, int w, int h, int workers, uint64_t* counts) {
    return guard([&] {
        Histogram hs = build_histogram(gray_in(gray, w, h), workers);
        for (int v = 0; v < 256; ++v) counts[v] = hs.counts[v];
    });
}

int ref_kmeans(const uint64_t* counts, int k, int max_iter, double tol, double* centers,
               uint16_t* assign, int* iters) {
    return guard([&] {
        Histogram hs;
        for (int v = 0; v < 256; ++v) hs.counts[v] = counts[v];
        Clustering c = kmeans_histogram(hs, k, max_iter, tol);
        for (int j = 0; j < c.k(); ++j) centers[j] = c.centers[j];
        for (int v = 0; v < 256; ++v) assign[v] = c.bin_assignment[v];
        *iters = c.iterations_run;
    });
}

int ref_detect(const uint16_t* labels, int w, int h, uint8_t* out) {
    return guard([&] {
        LabelMap lm(w, h);
        std::memcpy(lm.labels.data(), labels, lm.labels.size() * 2);
        BoundaryMask m = detect_boundaries(lm, 1);
        std::memcpy(out, m.mask.data(), m.mask.size());
    });
}

int ref_fill(const uint8_t* in, int w, int h, uint8_t* out) {
    return guard([&] {
        BoundaryMask m = morph_fill(mask_in(in, w, h), 1);
        std::memcpy(out, m.mask.data(), m.mask.size());
    });
}

int ref_remove(const uint8_t* in, int w, int h, uint8_t* out) {
    return guard([&] {
        BoundaryMask m = morph_remove(mask_in(in, w, h), 1);
        std::memcpy(out, m.mask.data(), m.mask.size());
    });
}

int ref_label_components(const uint8_t* in, int w, int h, int32_t* labels, uint32_t* sizes,
                         int32_t* by_size) {
    int n = -1;
    int rc = guard([&] {
        ComponentTable t = label_components(mask_in(in, w, h));
        std::memcpy(labels, t.labels.data(), t.labels.size() * 4);
        std::memcpy(sizes, t.sizes.data(), t.sizes.size() * 4);
        std::memcpy(by_size, t.by_size.data(), t.by_size.size() * 4);
        n = static_cast<int>(t.sizes.size());
    });
    return rc ? rc : n;
}

int ref_prune(const uint8_t* in, int w, int h, double fraction, uint8_t* out) {
    return guard([&] {
        BoundaryMask m = prune_components(mask_in(in, w, h), fraction);
        std::memcpy(out, m.mask.data(), m.mask.size());
    });
}

int ref_anchors(const uint8_t* in, int w, int h, int margin, uint8_t* out) {
    return guard([&] {
        BoundaryMask m = add_border_anchors(mask_in(in, w, h), margin);
        std::memcpy(out, m.mask.data(), m.mask.size());
    });
}

int ref_match(const uint8_t* l, const uint8_t* r, const uint8_t* mask, int w, int h,
              int window, int max_disparity, int workers, int16_t* out) {
    return guard([&] {
        MatchConfig mc{window, max_disparity};
        DisparityMap d = match_boundary_pixels(gray_in(l, w, h), gray_in(r, w, h),
                                               mask_in(mask, w, h), mc, workers);
        std::memcpy(out, d.values.data(), d.values.size() * 2);
    });
}

int ref_fill_scanlines(const int16_t* in, int w, int h, int16_t* out) {
    return guard([&] {
        DisparityMap d = fill_scanlines(disp_in(in, w, h), 1);
        std::memcpy(out, d.values.data(), d.values.size() * 2);
    });
}

int ref_peek_columns(const int16_t* in, int w, int h, int threshold, int16_t* out) {
    return guard([&] {
        DisparityMap d = peek_columns(disp_in(in, w, h), threshold, 1);
        std::memcpy(out, d.values.data(), d.values.size() * 2);
    });
}

int ref_gaussian_kernel(double sigma, int size, double* weights) {
    return guard([&] {
        GaussianKernel k = gaussian_kernel(sigma, size);
        std::memcpy(weights, k.weights.data(), k.weights.size() * 8);
    });
}

int ref_blur_map(const int16_t* depth, int w, int h, const int* lo, const int* hi, int n,
                 int max_disparity, uint8_t* out) {
    return guard([&] {
        FocusSpec f;
        for (int i = 0; i < n; ++i) f.ranges.emplace_back(lo[i], hi[i]);
        GrayImage m = build_blur_map(disp_in(depth, w, h), f, max_disparity);
        std::memcpy(out, m.data.data(), m.data.size());
    });
}

int ref_selective_blur(const uint8_t* rgb, const uint8_t* map, int w, int h, double sigma,
                       int size, int workers, uint8_t* out) {
    return guard([&] {
        GaussianKernel k = gaussian_kernel(sigma, size);
        RgbImage o = selective_blur(rgb_in(rgb, w, h), gray_in(map, w, h), k, workers);
        std::memcpy(out, o.data.data(), o.data.size());
    });
}

// Full frame through the reference's own run_depth_pipeline (with StageTimes)
// followed by build_blur_map + gaussian_kernel + selective_blur, i.e. exactly
// run_refocus_pipeline's work (pipeline.cpp:136-151) plus per-stage timing.
// times_ms[7] = convert, segment, boundary, match, fill, peek, blur.
// Any output pointer may be NULL.
int ref_run_frame(const uint8_t* rgb_l, const uint8_t* rgb_r, int w, int h, int k, int window,
                  int max_disparity, int threshold, double prune_fraction, int workers,
                  const int* lo, const int* hi, int n_ranges, double sigma, int kernel_size,
                  uint8_t* refocused, int16_t* dense, int16_t* sparse, uint8_t* gray_l,
                  uint8_t* gray_r, uint16_t* labels, uint8_t* braw, uint8_t* bref,
                  uint8_t* banc, int16_t* row_filled, double* centers, uint16_t* assign,
                  int* k_iters, uint64_t* stats4, double* frac2, double* times_ms) {
    return guard([&] {
        PipelineConfig cfg;
        cfg.k = k;
        cfg.window = window;
        cfg.max_disparity = max_disparity;
        cfg.threshold = threshold;
        cfg.prune_fraction = prune_fraction;
        cfg.workers = workers;
        RgbImage L = rgb_in(rgb_l, w, h), R = rgb_in(rgb_r, w, h);
        StageTimes t;
        DepthResult d = run_depth_pipeline(L, R, cfg, &t);
        double blur_ms = 0.0;
        if (refocused && n_ranges > 0) {
            auto t0 = std::chrono::steady_clock::now();
            FocusSpec f;
            for (int i = 0; i < n_ranges; ++i) f.ranges.emplace_back(lo[i], hi[i]);
            f.sigma = sigma;
            GrayImage map = build_blur_map(d.dense, f, max_disparity);
            const int size = kernel_size > 0 ? kernel_size : default_kernel_size(sigma);
            GaussianKernel kern = gaussian_kernel(sigma, size);
            RgbImage o = selective_blur(L, map, kern, workers);
            blur_ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0)
                          .count();
            std::memcpy(refocused, o.data.data(), o.data.size());
        }
        const size_t n = static_cast<size_t>(w) * h;
        if (dense) std::memcpy(dense, d.dense.values.data(), n * 2);
        if (sparse) std::memcpy(sparse, d.sparse.values.data(), n * 2);
        if (row_filled) std::memcpy(row_filled, d.row_filled.values.data(), n * 2);
        if (gray_l) std::memcpy(gray_l, d.left_lightness.data.data(), n);
        if (gray_r) std::memcpy(gray_r, d.right_lightness.data.data(), n);
        if (labels) std::memcpy(labels, d.labels.labels.data(), n * 2);
        if (braw) std::memcpy(braw, d.boundary_raw.mask.data(), n);
        if (bref) std::memcpy(bref, d.boundary_refined.mask.data(), n);
        if (banc) std::memcpy(banc, d.boundary_anchored.mask.data(), n);
        if (centers)
            for (int j = 0; j < d.clustering.k(); ++j) centers[j] = d.clustering.centers[j];
        if (assign)
            for (int v = 0; v < 256; ++v) assign[v] = d.clustering.bin_assignment[v];
        if (k_iters) {
            k_iters[0] = d.clustering.k();
            k_iters[1] = d.clustering.iterations_run;
        }
        if (stats4) {
            stats4[0] = d.stats.pixels;
            stats4[1] = d.stats.boundary_raw;
            stats4[2] = d.stats.boundary_refined;
            stats4[3] = d.stats.matched;
        }
        if (frac2) {
            frac2[0] = d.stats.matched_fraction;
            frac2[1] = d.stats.known_fraction;
        }
        if (times_ms) {
            times_ms[0] = t.convert;
            times_ms[1] = t.segment;
            times_ms[2] = t.boundary;
            times_ms[3] = t.match;
            times_ms[4] = t.fill;
            times_ms[5] = t.peek;
            times_ms[6] = blur_ms;
        }
    });
}

// The reference's own deterministic scene generators (tests/synthetic.cpp).
static void pair_out(const StereoPair& p, uint8_t* l, uint8_t* r) {
    std::memcpy(l, p.left.data.data(), p.left.data.size());
    std::memcpy(r, p.right.data.data(), p.right.data.size());
}
void ref_synth_bench_frame(int w, int h, uint32_t seed, uint8_t* l, uint8_t* r) {
    pair_out(synthetic::bench_frame(w, h, seed), l, r);
}
void ref_synth_rectangle_scene(int w, int h, int shift, uint32_t seed, uint8_t* l, uint8_t* r) {
    pair_out(synthetic::rectangle_scene_pair(w, h, shift, seed), l, r);
}
void ref_synth_translated_noise(int w, int h, int shift, uint32_t seed, uint8_t* l, uint8_t* r) {
    pair_out(synthetic::translated_noise_pair(w, h, shift, seed), l, r);
}
void ref_synth_random_rgb(int w, int h, uint32_t seed, uint8_t* out) {
    RgbImage im = synthetic::random_rgb(w, h, seed);
    std::memcpy(out, im.data.data(), im.data.size());
}
void ref_synth_random_gray(int w, int h, uint32_t seed, uint8_t* out) {
    GrayImage im = synthetic::random_gray(w, h, seed);
    std::memcpy(out, im.data.data(), im.data.size());
}
void ref_synth_random_mask(int w, int h, uint32_t seed, int percent, uint8_t* out) {
    BoundaryMask m = synthetic::random_mask(w, h, seed, percent);
    std::memcpy(out, m.mask.data(), m.mask.size());
}
void ref_synth_random_sparse(int w, int h, uint32_t seed, int percent, int dmax, int16_t* out) {
    DisparityMap d = synthetic::random_sparse(w, h, seed, percent, dmax);
    std::memcpy(out, d.values.data(), d.values.size() * 2);
}

int ref_hardware_workers() { return hardware_workers(); }

}  // extern "C"
