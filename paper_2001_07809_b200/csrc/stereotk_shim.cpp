// stereotk_shim.cpp -- the reference's stereotk:: C++ API (value types,
// exceptions) implemented on the C-ABI of stk_b200.h.  One implicit context
// per host thread (device from stereotk::b200::set_device or $STK_DEVICE).
// STK_EPARAM becomes stereotk::ParamError with the C-ABI's message (which
// mirrors the reference's text); any other failure becomes std::runtime_error.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <sstream>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <cstdio>
#include <string>

#include "stereotk/stereotk_b200.hpp"
#include "stk_b200.h"

namespace stereotk {

namespace {

struct CtxHolder {
    stk_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) stk_destroy(ctx);
    }
};

thread_local CtxHolder t_ctx;
thread_local int t_device = -1;
thread_local bool t_fast_blur = true;

void check(stk_status s, const stk_ctx* ctx) {
    if (s == STK_OK) return;
    const std::string msg = stk_last_error(ctx);
    switch (s) {
        case STK_EPARAM: throw ParamError(msg);
        case STK_EIO: throw IoError(msg);
        case STK_EFORMAT: throw FormatError(msg);
        default: throw std::runtime_error(msg);
    }
}

stk_ctx* ctx() {
    int dev = t_device;
    if (dev < 0) {
        const char* e = std::getenv("STK_DEVICE");
        dev = e ? std::atoi(e) : 0;
    }
    if (!t_ctx.ctx || t_ctx.device != dev) {
        if (t_ctx.ctx) stk_destroy(t_ctx.ctx);
        t_ctx.ctx = nullptr;
        stk_ctx* c = nullptr;
        check(stk_create(dev, 0, 0, 1, &c), nullptr);
        t_ctx.ctx = c;
        t_ctx.device = dev;
    }
    return t_ctx.ctx;
}

void check_workers(int workers) {
    (void)workers;  // any value: results are identical (parallel.hpp:24-28)
}

std::string dims(int w, int h) { return std::to_string(w) + "x" + std::to_string(h); }

}  // namespace

namespace b200 {
void set_device(int device) { t_device = device; }
void set_fast_blur(bool on) { t_fast_blur = on; }
bool fast_blur() { return t_fast_blur; }
}  // namespace b200

GrayImage rgb_to_lightness(const RgbImage& image, int workers) {
    check_workers(workers);
    GrayImage out(image.width, image.height);
    stk_ctx* c = ctx();
    check(stk_rgb_to_lightness(c, image.data.data(), image.width, image.height, out.data.data()), c);
    return out;
}

Histogram build_histogram(const GrayImage& image, int workers) {
    check_workers(workers);
    Histogram h;
    stk_ctx* c = ctx();
    check(stk_build_histogram(c, image.data.data(), image.width, image.height, h.counts.data()), c);
    return h;
}

Clustering kmeans_histogram(const Histogram& histogram, int k, int max_iter, double tol) {
    Clustering cl;
    std::vector<double> centers(k > 0 ? k : 1);
    int iters = 0;
    stk_ctx* c = ctx();
    check(stk_kmeans_histogram(c, histogram.counts.data(), k, max_iter, tol, centers.data(),
                               cl.bin_assignment.data(), &iters),
          c);
    centers.resize(k);
    cl.centers = std::move(centers);
    cl.iterations_run = iters;
    return cl;
}

LabelMap assign_pixels(const GrayImage& image, const Clustering& clustering) {
    LabelMap out(image.width, image.height);
    stk_ctx* c = ctx();
    check(stk_assign_pixels(c, image.data.data(), image.width, image.height,
                            clustering.bin_assignment.data(), clustering.k(), out.labels.data()),
          c);
    return out;
}

BoundaryMask detect_boundaries(const LabelMap& labels, int workers) {
    check_workers(workers);
    BoundaryMask out(labels.width, labels.height);
    stk_ctx* c = ctx();
    check(stk_detect_boundaries(c, labels.labels.data(), labels.width, labels.height, out.mask.data()), c);
    return out;
}

BoundaryMask morph_fill(const BoundaryMask& mask, int workers) {
    check_workers(workers);
    BoundaryMask out(mask.width, mask.height);
    stk_ctx* c = ctx();
    check(stk_morph_fill(c, mask.mask.data(), mask.width, mask.height, out.mask.data()), c);
    return out;
}

BoundaryMask morph_remove(const BoundaryMask& mask, int workers) {
    check_workers(workers);
    BoundaryMask out(mask.width, mask.height);
    stk_ctx* c = ctx();
    check(stk_morph_remove(c, mask.mask.data(), mask.width, mask.height, out.mask.data()), c);
    return out;
}

ComponentTable label_components(const BoundaryMask& mask) {
    ComponentTable t;
    t.width = mask.width;
    t.height = mask.height;
    const std::size_t n = mask.mask.size();
    t.labels.assign(n, -1);
    std::vector<std::uint32_t> sizes(n ? n : 1);
    std::vector<std::int32_t> bys(n ? n : 1);
    int nc = 0;
    stk_ctx* c = ctx();
    check(stk_label_components(c, mask.mask.data(), mask.width, mask.height, t.labels.data(),
                               sizes.data(), bys.data(), sizes.size(), &nc),
          c);
    sizes.resize(nc);
    bys.resize(nc);
    t.sizes = std::move(sizes);
    t.by_size = std::move(bys);
    return t;
}

BoundaryMask prune_components(const BoundaryMask& mask, double fraction) {
    BoundaryMask out(mask.width, mask.height);
    stk_ctx* c = ctx();
    check(stk_prune_components(c, mask.mask.data(), mask.width, mask.height, fraction, out.mask.data()), c);
    return out;
}

BoundaryMask add_border_anchors(const BoundaryMask& mask, int margin) {
    BoundaryMask out(mask.width, mask.height);
    stk_ctx* c = ctx();
    check(stk_add_border_anchors(c, mask.mask.data(), mask.width, mask.height, margin, out.mask.data()),
          c);
    return out;
}

std::uint32_t sad_cost(const GrayImage& left, const GrayImage& right, int x, int y, int d, int window) {
    std::uint32_t cost = 0;
    stk_ctx* c = ctx();
    check(stk_sad_cost(c, left.data.data(), right.data.data(), left.width, left.height, x, y, d, window,
                       &cost),
          c);
    return cost;
}

DisparityMap match_boundary_pixels(const GrayImage& left, const GrayImage& right,
                                   const BoundaryMask& mask, const MatchConfig& config, int workers) {
    check_workers(workers);
    if (left.width != right.width || left.height != right.height)  // stereo.cpp:36-43
        throw ParamError("stereo: image sizes differ, left " + dims(left.width, left.height) +
                         " vs right " + dims(right.width, right.height));
    if (mask.width != left.width || mask.height != left.height)
        throw ParamError("stereo: mask size " + dims(mask.width, mask.height) +
                         " does not match images " + dims(left.width, left.height));
    DisparityMap out(left.width, left.height);
    stk_ctx* c = ctx();
    check(stk_match_boundary_pixels(c, left.data.data(), right.data.data(), mask.mask.data(), left.width,
                                    left.height, config.window, config.max_disparity, out.values.data()),
          c);
    return out;
}

EvalResult bad_pixel_rate(const DisparityMap& computed, const DisparityMap& truth, double delta_d,
                          int workers) {
    check_workers(workers);
    if (computed.width != truth.width || computed.height != truth.height)  // evaluate.cpp:20-26
        throw ParamError("bad_pixel_rate: computed " + dims(computed.width, computed.height) +
                         " vs truth " + dims(truth.width, truth.height));
    EvalResult r;
    r.delta_d = delta_d;
    stk_ctx* c = ctx();
    check(stk_bad_pixel_rate(c, computed.values.data(), truth.values.data(), computed.width,
                             computed.height, delta_d, &r.bad_pixel_rate, &r.compared, &r.excluded),
          c);
    return r;
}

DisparityMap dense_sad_baseline(const GrayImage& left, const GrayImage& right,
                                const MatchConfig& config, int workers) {
    check_workers(workers);
    if (left.width != right.width || left.height != right.height)  // evaluate.cpp:95-101
        throw ParamError("dense_sad_baseline: image sizes differ, left " + dims(left.width, left.height) +
                         " vs right " + dims(right.width, right.height));
    DisparityMap out(left.width, left.height);
    stk_ctx* c = ctx();
    check(stk_dense_sad_baseline(c, left.data.data(), right.data.data(), left.width, left.height,
                                 config.window, config.max_disparity, out.values.data()),
          c);
    return out;
}

// bench.cpp:13-108 over the GPU pipeline.
namespace {
StageTimes measure_batch(const std::vector<StereoPair>& frames, const PipelineConfig& config) {
    StageTimes scratch;  // warm-up (bench.cpp:15-20)
    run_depth_pipeline(frames.front().left, frames.front().right, config, &scratch);
    StageTimes total;
    for (const StereoPair& frame : frames) {
        StageTimes t;
        run_depth_pipeline(frame.left, frame.right, config, &t);
        total.convert += t.convert;
        total.segment += t.segment;
        total.boundary += t.boundary;
        total.match += t.match;
        total.fill += t.fill;
        total.peek += t.peek;
    }
    return total;
}
}  // namespace

std::vector<BenchReport> run_benchmark(const std::vector<StereoPair>& frames,
                                       const std::vector<int>& worker_counts,
                                       const PipelineConfig& config) {
    if (frames.empty()) throw ParamError("benchmark: no frames given");
    if (worker_counts.empty()) throw ParamError("benchmark: no worker counts given");
    if (std::find(worker_counts.begin(), worker_counts.end(), 1) == worker_counts.end())
        throw ParamError("benchmark: worker counts must include 1, the serial baseline");
    for (int w : worker_counts)
        if (w < 1) throw ParamError("benchmark: worker count must be >= 1, got " + std::to_string(w));
    PipelineConfig serial_config = config;
    serial_config.workers = 1;
    const StageTimes serial = measure_batch(frames, serial_config);
    std::vector<BenchReport> reports;
    for (int workers : worker_counts) {
        BenchReport r;
        r.workers = workers;
        r.frames = static_cast<int>(frames.size());
        r.serial = serial;
        if (workers == 1) {
            r.times = serial;
        } else {
            PipelineConfig run_config = config;
            run_config.workers = workers;
            r.times = measure_batch(frames, run_config);
        }
        r.speedup = r.times.total() > 0.0 ? serial.total() / r.times.total() : 0.0;
        reports.push_back(r);
    }
    return reports;
}

std::string benchmark_csv(const std::vector<BenchReport>& reports) {
    std::ostringstream out;
    out << "frames,workers,stage,serial_ms,parallel_ms,speedup\n";
    auto row = [&](int f, int w, const char* stage, double s, double p) {
        out << f << ',' << w << ',' << stage << ',' << s << ',' << p << ',' << (p > 0.0 ? s / p : 0.0)
            << '\n';
    };
    for (const BenchReport& r : reports) {
        const StageTimes& s = r.serial;
        const StageTimes& t = r.times;
        row(r.frames, r.workers, "convert", s.convert, t.convert);
        row(r.frames, r.workers, "segment", s.segment, t.segment);
        row(r.frames, r.workers, "boundary", s.boundary, t.boundary);
        row(r.frames, r.workers, "match", s.match, t.match);
        row(r.frames, r.workers, "fill", s.fill, t.fill);
        row(r.frames, r.workers, "peek", s.peek, t.peek);
        row(r.frames, r.workers, "total", s.total(), t.total());
    }
    return out.str();
}

// --------------------------------------------- GPU-count benchmark axis --
namespace {

uint64_t fnv1a(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

struct GpuShare {  // one GPU's part of a batch
    StageTimes t;
    double blur = 0.0;
    std::array<double, 7> bytes{};
    std::vector<std::pair<int, uint64_t>> digests;
    std::string err;
    int err_code = 0;
};

struct StartGate {  // every GPU warmed up before the clock starts
    std::mutex m;
    std::condition_variable cv;
    int ready = 0;
    bool go = false;
};

// GPU g of G: frames g, g + G, ... on two slots of its own context.
void gpu_share(int g, int G, int device, const std::vector<StereoPair>& frames, const stk_config& cfg,
               const stk_focus* fo, StartGate& gate, GpuShare& out) {
    stk_ctx* c = nullptr;
    auto fail = [&](stk_status st) {
        out.err_code = st;
        out.err = stk_last_error(c);
    };
    const int w = frames.front().left.width, h = frames.front().left.height;
    stk_status st = stk_create(device, w, h, 2, &c);
    struct Buf {
        std::vector<int16_t> dense;
        std::vector<uint8_t> rgb;
        int frame = -1;
    } buf[2];
    if (st == STK_OK) {  // warm-up (bench.cpp:15-20): one untimed frame
        for (Buf& b : buf) {
            b.dense.resize((size_t)w * h);
            b.rgb.resize(fo ? (size_t)w * h * 3 : 0);
        }
        stk_frame_out o{};
        o.dense = buf[0].dense.data();
        o.refocused = fo ? buf[0].rgb.data() : nullptr;
        const StereoPair& p = frames[g % frames.size()];
        st = stk_frame_submit(c, 0, p.left.data.data(), p.right.data.data(), w, h, &cfg, fo, &o, 1);
        if (st == STK_OK) st = stk_frame_wait(c, 0, nullptr, nullptr, nullptr);
    }
    if (st != STK_OK) fail(st);
    {
        std::unique_lock<std::mutex> lk(gate.m);
        ++gate.ready;
        gate.cv.notify_all();
        gate.cv.wait(lk, [&] { return gate.go; });
    }
    const double N = (double)w * h;
    auto collect = [&](int slot) -> stk_status {
        stk_stats sst{};
        stk_times tm{};
        const stk_status r = stk_frame_wait(c, slot, &sst, &tm, nullptr);
        if (r != STK_OK) return r;
        out.t.convert += tm.convert;
        out.t.segment += tm.segment;
        out.t.boundary += tm.boundary;
        out.t.match += tm.match;
        out.t.fill += tm.fill;
        out.t.peek += tm.peek;
        out.blur += tm.blur;
        const double M = (double)sst.matched;
        const double b[7] = {8 * N, N, 12 * N + 4 * M, 4 * N + 4 * M, 4 * N, 4 * N, fo ? 8 * N : 0.0};
        for (int i = 0; i < 7; ++i) out.bytes[i] += b[i];
        Buf& bb = buf[slot];
        uint64_t dg = fnv1a(bb.dense.data(), bb.dense.size() * 2);
        if (fo) dg = fnv1a(bb.rgb.data(), bb.rgb.size(), dg);
        out.digests.emplace_back(bb.frame, dg);
        bb.frame = -1;
        return STK_OK;
    };
    if (st == STK_OK) {
        int k = 0;
        for (size_t f = g; f < frames.size() && st == STK_OK; f += G, ++k) {
            const int slot = k & 1;
            if (buf[slot].frame >= 0 && (st = collect(slot)) != STK_OK) break;
            stk_frame_out o{};
            o.dense = buf[slot].dense.data();
            o.refocused = fo ? buf[slot].rgb.data() : nullptr;
            const StereoPair& p = frames[f];
            st = stk_frame_submit(c, slot, p.left.data.data(), p.right.data.data(), w, h, &cfg, fo, &o, 1);
            if (st == STK_OK) buf[slot].frame = (int)f;
        }
        for (int slot = 0; slot < 2 && st == STK_OK; ++slot)
            if (buf[slot].frame >= 0) st = collect(slot);
        if (st != STK_OK) fail(st);
    }
    if (c) stk_destroy(c);
}

struct BatchResult {
    StageTimes t;       // max over GPUs of the per-GPU stage sums
    double blur = 0.0;
    double wall_ms = 0.0;
    std::array<double, 7> bytes{};
    std::vector<uint64_t> digests;
};

BatchResult gpu_batch(const std::vector<StereoPair>& frames, int G, const stk_config& cfg,
                      const stk_focus* fo) {
    const int ndev = std::max(1, stk_device_count());
    std::vector<GpuShare> shares(G);
    StartGate gate;
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
        th.emplace_back(gpu_share, g, G, g % ndev, std::cref(frames), std::cref(cfg), fo, std::ref(gate),
                        std::ref(shares[g]));
    std::chrono::steady_clock::time_point t0;
    {
        std::unique_lock<std::mutex> lk(gate.m);
        gate.cv.wait(lk, [&] { return gate.ready == G; });
        t0 = std::chrono::steady_clock::now();
        gate.go = true;
        gate.cv.notify_all();
    }
    for (auto& t : th) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    BatchResult r;
    r.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    r.digests.assign(frames.size(), 0);
    for (const GpuShare& s : shares) {
        if (s.err_code) {
            if (s.err_code == STK_EPARAM) throw ParamError(s.err);
            throw std::runtime_error(s.err);
        }
        r.t.convert = std::max(r.t.convert, s.t.convert);
        r.t.segment = std::max(r.t.segment, s.t.segment);
        r.t.boundary = std::max(r.t.boundary, s.t.boundary);
        r.t.match = std::max(r.t.match, s.t.match);
        r.t.fill = std::max(r.t.fill, s.t.fill);
        r.t.peek = std::max(r.t.peek, s.t.peek);
        r.blur = std::max(r.blur, s.blur);
        for (int i = 0; i < 7; ++i) r.bytes[i] += s.bytes[i];
        for (const auto& d : s.digests) r.digests[d.first] = d.second;
    }
    return r;
}

}  // namespace

std::vector<GpuBenchReport> run_benchmark_gpus(const std::vector<StereoPair>& frames,
                                               const std::vector<int>& gpu_counts,
                                               const PipelineConfig& config, const FocusSpec* focus,
                                               int kernel_size) {
    if (frames.empty()) throw ParamError("benchmark: no frames given");
    if (gpu_counts.empty()) throw ParamError("benchmark: no GPU counts given");
    if (std::find(gpu_counts.begin(), gpu_counts.end(), 1) == gpu_counts.end())
        throw ParamError("benchmark: GPU counts must include 1, the single-GPU baseline");
    for (int g : gpu_counts)
        if (g < 1) throw ParamError("benchmark: GPU count must be >= 1, got " + std::to_string(g));
    validate_config(config);
    for (const StereoPair& p : frames)
        if (!p.left.same_size(p.right) || !p.left.same_size(frames.front().left))
            throw ParamError("benchmark: frames differ in size, " + dims(p.left.width, p.left.height) +
                             " vs " + dims(frames.front().left.width, frames.front().left.height));
    const stk_config cfg{config.k, config.window, config.max_disparity, config.threshold,
                         config.prune_fraction, config.workers};
    std::vector<int> lo, hi;
    stk_focus fo{};
    if (focus) {
        for (const auto& r : focus->ranges) {
            lo.push_back(r.first);
            hi.push_back(r.second);
        }
        fo = stk_focus{lo.data(), hi.data(), static_cast<int>(lo.size()), focus->sigma, kernel_size,
                       t_fast_blur ? 0 : 1};
    }
    const BatchResult serial = gpu_batch(frames, 1, cfg, focus ? &fo : nullptr);
    std::vector<GpuBenchReport> reports;
    for (int G : gpu_counts) {
        const BatchResult b = G == 1 ? serial : gpu_batch(frames, G, cfg, focus ? &fo : nullptr);
        GpuBenchReport r;
        r.gpus = G;
        r.frames = static_cast<int>(frames.size());
        r.times = b.t;
        r.blur = b.blur;
        r.serial = serial.t;
        r.serial_blur = serial.blur;
        r.wall_ms = b.wall_ms;
        r.serial_wall_ms = serial.wall_ms;
        r.frames_per_s = b.wall_ms > 0.0 ? 1e3 * r.frames / b.wall_ms : 0.0;
        r.speedup = b.wall_ms > 0.0 ? serial.wall_ms / b.wall_ms : 0.0;
        r.alg_bytes = b.bytes;
        r.digests = b.digests;
        reports.push_back(std::move(r));
    }
    return reports;
}

std::string benchmark_csv(const std::vector<GpuBenchReport>& reports) {
    std::ostringstream out;
    out << "frames,gpus,stage,serial_ms,parallel_ms,speedup,alg_bytes,gb_per_s\n";
    auto row = [&](const GpuBenchReport& r, const char* stage, double s, double p, double bytes) {
        out << r.frames << ',' << r.gpus << ',' << stage << ',' << s << ',' << p << ','
            << (p > 0.0 ? s / p : 0.0) << ',' << bytes << ',' << (p > 0.0 ? bytes / (p * 1e-3) / 1e9 : 0.0)
            << '\n';
    };
    for (const GpuBenchReport& r : reports) {
        const StageTimes& s = r.serial;
        const StageTimes& t = r.times;
        const auto& b = r.alg_bytes;
        row(r, "convert", s.convert, t.convert, b[0]);
        row(r, "segment", s.segment, t.segment, b[1]);
        row(r, "boundary", s.boundary, t.boundary, b[2]);
        row(r, "match", s.match, t.match, b[3]);
        row(r, "fill", s.fill, t.fill, b[4]);
        row(r, "peek", s.peek, t.peek, b[5]);
        row(r, "blur", r.serial_blur, r.blur, b[6]);
        double tot = 0.0;
        for (double v : b) tot += v;
        row(r, "total", r.serial_wall_ms, r.wall_ms, tot);
    }
    return out.str();
}

// evaluate.cpp:220-227: nlohmann::json dump -- keys in sorted order, compact.
std::string eval_report_json(const EvalResult& r) {
    return "{\"bad_pixel_rate\":" + b200::json_number(r.bad_pixel_rate) + ",\"compared\":" +
           std::to_string(r.compared) + ",\"delta_d\":" + b200::json_number(r.delta_d) +
           ",\"excluded\":" + std::to_string(r.excluded) + "}";
}

// nlohmann::json's double serialisation: the shortest digit string that
// round-trips, laid out as its format_buffer does (decimal point kept for
// integral values, plain notation for decimal exponents in (-4, 15], else
// d.ddde+XX with at least two exponent digits).
std::string b200::json_number(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    int p = 1;
    for (; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*e", p - 1, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf, sign;
    if (s[0] == '-') {
        sign = "-";
        s.erase(0, 1);
    }
    const std::size_t e = s.find('e');
    const int exp10 = std::atoi(s.c_str() + e + 1);
    std::string digits;
    for (std::size_t i = 0; i < e; ++i)
        if (s[i] != '.') digits += s[i];
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(-n, '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
        out += eb;
    }
    return sign + out;
}

DisparityMap fill_scanlines(const DisparityMap& sparse, int workers) {
    check_workers(workers);
    DisparityMap out(sparse.width, sparse.height);
    stk_ctx* c = ctx();
    check(stk_fill_scanlines(c, sparse.values.data(), sparse.width, sparse.height, out.values.data()), c);
    return out;
}

DisparityMap peek_columns(const DisparityMap& map, int threshold, int workers) {
    check_workers(workers);
    DisparityMap out(map.width, map.height);
    stk_ctx* c = ctx();
    check(stk_peek_columns(c, map.values.data(), map.width, map.height, threshold, out.values.data()), c);
    return out;
}

int default_kernel_size(double sigma) { return stk_default_kernel_size(sigma); }

GaussianKernel gaussian_kernel(double sigma, int size) {
    GaussianKernel k;
    k.size = size;
    k.weights.assign(size > 0 ? static_cast<std::size_t>(size) * size : 0, 0.0);
    check(stk_gaussian_kernel(sigma, size, k.weights.data()), nullptr);
    return k;
}

GrayImage build_blur_map(const DisparityMap& depth, const FocusSpec& focus, int max_disparity) {
    std::vector<int> lo, hi;
    for (const auto& r : focus.ranges) {
        lo.push_back(r.first);
        hi.push_back(r.second);
    }
    GrayImage out(depth.width, depth.height);
    stk_ctx* c = ctx();
    check(stk_build_blur_map(c, depth.values.data(), depth.width, depth.height, lo.data(), hi.data(),
                             static_cast<int>(lo.size()), max_disparity, out.data.data()),
          c);
    return out;
}

namespace {
// sigma such that the kernel is exactly gaussian_kernel(sigma, size), or 0
double gaussian_sigma_of(const GaussianKernel& k) {
    if (k.size < 3) return 0.0;
    const int h = k.size / 2;
    const double r = k.at(0, 1) / k.at(0, 0);
    if (!(r > 0.0 && r < 1.0)) return 0.0;
    const double sigma = std::sqrt(-1.0 / (2.0 * std::log(r)));
    for (double cand : {sigma, std::nextafter(sigma, 0.0), std::nextafter(sigma, 1e300)}) {
        std::vector<double> w(static_cast<std::size_t>(k.size) * k.size);
        if (stk_gaussian_kernel(cand, k.size, w.data()) != STK_OK) continue;
        if (std::memcmp(w.data(), k.weights.data(), w.size() * sizeof(double)) == 0) return cand;
    }
    (void)h;
    return 0.0;
}
}  // namespace

RgbImage selective_blur(const RgbImage& image, const GrayImage& blur_map, const GaussianKernel& kernel,
                        int workers) {
    check_workers(workers);
    if (blur_map.width != image.width || blur_map.height != image.height)  // refocus.cpp:77-84
        throw ParamError("selective_blur: blur map " + dims(blur_map.width, blur_map.height) +
                         " does not match image " + dims(image.width, image.height));
    RgbImage out(image.width, image.height);
    stk_ctx* c = ctx();
    const double sigma = t_fast_blur ? gaussian_sigma_of(kernel) : 0.0;
    if (sigma > 0.0)
        check(stk_selective_blur(c, image.data.data(), blur_map.data.data(), image.width, image.height,
                                 sigma, kernel.size, 0, out.data.data()),
              c);
    else
        check(stk_selective_blur_weights(c, image.data.data(), blur_map.data.data(), image.width,
                                         image.height, kernel.weights.data(), kernel.size,
                                         out.data.data()),
              c);
    return out;
}

void validate_config(const PipelineConfig& config) {
    const stk_config cfg{config.k, config.window, config.max_disparity, config.threshold,
                         config.prune_fraction, config.workers};
    check(stk_validate_config(&cfg), nullptr);
}

namespace {
RgbImage run_frame(const RgbImage& left, const RgbImage& right, const PipelineConfig& config,
                   const FocusSpec* focus, int kernel_size, DepthResult* depth, StageTimes* times) {
    validate_config(config);
    if (!left.same_size(right))  // pipeline.cpp:54-60
        throw ParamError("pipeline: image sizes differ, left " + dims(left.width, left.height) +
                         " vs right " + dims(right.width, right.height));
    const int w = left.width, h = left.height;
    const stk_config cfg{config.k, config.window, config.max_disparity, config.threshold,
                         config.prune_fraction, config.workers};
    std::vector<int> lo, hi;
    stk_focus fo{};
    if (focus) {
        for (const auto& r : focus->ranges) {
            lo.push_back(r.first);
            hi.push_back(r.second);
        }
        fo = stk_focus{lo.data(), hi.data(), static_cast<int>(lo.size()), focus->sigma, kernel_size,
                       t_fast_blur ? 0 : 1};
    }
    RgbImage out;
    DepthResult local;
    DepthResult& d = depth ? *depth : local;
    d.dense = DisparityMap(w, h);
    stk_frame_out o{};
    o.dense = d.dense.values.data();
    if (focus) {
        out = RgbImage(w, h);
        o.refocused = out.data.data();
    }
    double centers[256];
    if (depth) {
        d.left_lightness = GrayImage(w, h);
        d.right_lightness = GrayImage(w, h);
        d.labels = LabelMap(w, h);
        d.boundary_raw = BoundaryMask(w, h);
        d.boundary_refined = BoundaryMask(w, h);
        d.boundary_anchored = BoundaryMask(w, h);
        d.sparse = DisparityMap(w, h);
        d.row_filled = DisparityMap(w, h);
        o.left_lightness = d.left_lightness.data.data();
        o.right_lightness = d.right_lightness.data.data();
        o.labels = d.labels.labels.data();
        o.boundary_raw = d.boundary_raw.mask.data();
        o.boundary_refined = d.boundary_refined.mask.data();
        o.boundary_anchored = d.boundary_anchored.mask.data();
        o.sparse = d.sparse.values.data();
        o.row_filled = d.row_filled.values.data();
        o.centers = centers;
        o.bin_assignment = d.clustering.bin_assignment.data();
    }
    stk_ctx* c = ctx();
    stk_stats st{};
    stk_times tm{};
    stk_frame_info info{};
    check(stk_frame_submit(c, 0, left.data.data(), right.data.data(), w, h, &cfg, focus ? &fo : nullptr,
                           &o, times != nullptr),
          c);
    check(stk_frame_wait(c, 0, &st, &tm, &info), c);
    d.stats = DepthStats{st.pixels, st.boundary_raw, st.boundary_refined, st.matched,
                         st.matched_fraction, st.known_fraction};
    if (depth) {
        d.clustering.centers.assign(centers, centers + info.k);
        d.clustering.iterations_run = info.iterations_run;
    }
    if (times) {
        times->convert = tm.convert;
        times->segment = tm.segment;
        times->boundary = tm.boundary;
        times->match = tm.match;
        times->fill = tm.fill;
        times->peek = tm.peek;
    }
    return out;
}
}  // namespace

DepthResult run_depth_pipeline(const RgbImage& left, const RgbImage& right, const PipelineConfig& config,
                               StageTimes* times) {
    DepthResult d;
    run_frame(left, right, config, nullptr, 0, &d, times);
    return d;
}

RgbImage run_refocus_pipeline(const RgbImage& left, const RgbImage& right, const PipelineConfig& config,
                              const FocusSpec& focus, int kernel_size, DepthResult* depth_out) {
    return run_frame(left, right, config, &focus, kernel_size, depth_out, nullptr);
}

}  // namespace stereotk
