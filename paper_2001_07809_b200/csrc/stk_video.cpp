// stk_video.cpp -- a directory of stereo frame pairs through the GPU pipeline
// with file decode, PCIe copies, kernels and file encode all overlapped
// ("pinned, async decode overlapping H2D"; the paper's
// workload is a stereo video processed frame by frame).
//
// The reference has no such driver: its CLI refocuses one pair per process
// (tools/main.cpp:327-379) and `bench` loads every frame before timing
// (main.cpp:412-418).  Here frames stream:
//
//   decoder threads --> host buffer set (pinned) --> GPU slot (H2D, kernels,
//   D2H on the slot's stream) --> writer threads --> <out>/<stem>.<ext>
//
//   * H = slots + decoders + writers pinned host sets; frame f uses set f % H,
//     so decoders run up to H - slots frames ahead of the GPU;
//   * the main thread submits in frame order on GPU slot f % slots
//     (stk_frame_submit) and retires frame f - slots (stk_frame_wait) before
//     reusing its slot, handing the finished set to the writers;
//   * frames shard across processes / GPUs by index (f % shard_count ==
//     shard_index), the same frame -> rank rule as bench.py.
// Per frame the output is run_refocus_pipeline's image (and optionally the
// dense disparity via save_disparity), bit-identical to stk_run_frame.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <filesystem>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "stereotk/stereotk_b200.hpp"
#include "stk_b200.h"

namespace stk {
void set_thread_error(const std::string& msg);  // stk_capi.cu
}

namespace {

namespace fs = std::filesystem;
using stereotk::FormatError;
using stereotk::IoError;
using stereotk::ParamError;

struct HostSet {
    enum State { FREE, DECODING, DECODED, ON_GPU, WRITING };
    State state = FREE;
    int frame = -1;
    int w = 0, h = 0;
    std::size_t cap_px = 0;
    std::uint8_t *left = nullptr, *right = nullptr, *out = nullptr;
    std::int16_t* dense = nullptr;
};

struct Pipeline {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<HostSet> sets;
    std::string first_error;
    stk_status first_status = STK_OK;
    bool abort = false;

    void fail(stk_status s, const std::string& msg) {
        std::lock_guard<std::mutex> g(mu);
        if (first_status == STK_OK) {
            first_status = s;
            first_error = msg;
        }
        abort = true;
        cv.notify_all();
    }
};

stk_status classify(const std::exception& e) {
    if (dynamic_cast<const ParamError*>(&e)) return STK_EPARAM;
    if (dynamic_cast<const IoError*>(&e)) return STK_EIO;
    if (dynamic_cast<const FormatError*>(&e)) return STK_EFORMAT;
    return STK_EINTERNAL;
}

void ensure_pinned(HostSet& s, std::size_t px, bool dense) {
    if (s.cap_px >= px) return;
    stk_host_free(s.left);
    stk_host_free(s.right);
    stk_host_free(s.out);
    stk_host_free(s.dense);
    s.left = s.right = s.out = nullptr;
    s.dense = nullptr;
    void* p = nullptr;
    auto alloc = [&](std::size_t bytes) {
        if (stk_host_alloc(bytes, &p) != STK_OK) throw std::runtime_error("pinned host allocation failed");
        return p;
    };
    s.left = static_cast<std::uint8_t*>(alloc(px * 3));
    s.right = static_cast<std::uint8_t*>(alloc(px * 3));
    s.out = static_cast<std::uint8_t*>(alloc(px * 3));
    if (dense) s.dense = static_cast<std::int16_t*>(alloc(px * 2));
    s.cap_px = px;
}

std::string stem_of(const std::string& left_path) {
    std::string n = fs::path(left_path).filename().string();
    const std::size_t cut = n.rfind("_L.");
    return cut == std::string::npos ? n : n.substr(0, cut);
}

}  // namespace

extern "C" stk_status stk_video_refocus(stk_ctx* ctx, const char* in_dir, const char* out_dir,
                                        const stk_config* cfg, const stk_focus* focus,
                                        const stk_video_opts* opts, stk_video_report* report) {
    using clock = std::chrono::steady_clock;
    if (!ctx || !in_dir || !out_dir || !cfg || !focus || !opts) {
        stk::set_thread_error("stk_video_refocus: null argument");
        return STK_EPARAM;
    }
    const int slots = std::max(1, opts->slots);
    const int decoders = std::max(1, opts->decode_threads);
    const int writers = std::max(1, opts->write_threads);
    const int shard_n = std::max(1, opts->shard_count);
    const int shard_i = opts->shard_index;
    if (shard_i < 0 || shard_i >= shard_n) {
        stk::set_thread_error("stk_video_refocus: shard_index out of range");
        return STK_EPARAM;
    }
    std::vector<std::pair<std::string, std::string>> all;
    try {
        if (stk_status s = stk_validate_config(cfg); s != STK_OK) return s;
        all = stereotk::list_frame_pairs(in_dir);
        fs::create_directories(out_dir);
    } catch (const std::exception& e) {
        stk::set_thread_error(e.what());
        return classify(e);
    }
    std::vector<std::pair<std::string, std::string>> frames;
    for (std::size_t f = 0; f < all.size(); ++f)
        if (static_cast<int>(f % shard_n) == shard_i) frames.push_back(all[f]);
    const int n = static_cast<int>(frames.size());
    const std::string ext = opts->png ? ".png" : ".ppm";
    const bool want_dense = opts->disparity_scale > 0.0;

    Pipeline P;
    const int H = slots + decoders + writers;
    P.sets.resize(std::min(H, std::max(n, 1)));
    const int nsets = static_cast<int>(P.sets.size());
    std::atomic<int> next_decode{0};
    std::vector<int> write_queue;
    std::size_t qhead = 0;
    bool writers_done = false;
    double decode_s = 0.0, write_s = 0.0;
    std::mutex acc_mu;
    std::uint64_t matched = 0, pixels = 0;

    const auto t0 = clock::now();
    std::vector<std::thread> threads;
    for (int t = 0; t < decoders; ++t) {
        threads.emplace_back([&] {
            for (;;) {
                const int f = next_decode.fetch_add(1);
                if (f >= n) return;
                HostSet& s = P.sets[f % nsets];
                {
                    std::unique_lock<std::mutex> lk(P.mu);
                    P.cv.wait(lk, [&] { return P.abort || (s.state == HostSet::FREE && s.frame == (f < nsets ? -1 : f - nsets)); });
                    if (P.abort) return;
                    s.state = HostSet::DECODING;
                }
                const auto a = clock::now();
                try {
                    const stereotk::RgbImage l = stereotk::load_image(frames[f].first);
                    const stereotk::RgbImage r = stereotk::load_image(frames[f].second);
                    if (!l.same_size(r))  // pipeline.cpp:54-60
                        throw ParamError("pipeline: image sizes differ, left " + std::to_string(l.width) + "x" +
                                         std::to_string(l.height) + " vs right " + std::to_string(r.width) +
                                         "x" + std::to_string(r.height) + " (" + frames[f].first + ")");
                    ensure_pinned(s, l.pixel_count(), want_dense);
                    std::memcpy(s.left, l.data.data(), l.data.size());
                    std::memcpy(s.right, r.data.data(), r.data.size());
                    s.w = l.width;
                    s.h = l.height;
                } catch (const std::exception& e) {
                    P.fail(classify(e), e.what());
                    return;
                }
                {
                    std::lock_guard<std::mutex> g(acc_mu);
                    decode_s += std::chrono::duration<double>(clock::now() - a).count();
                }
                std::lock_guard<std::mutex> g(P.mu);
                s.frame = f;
                s.state = HostSet::DECODED;
                P.cv.notify_all();
            }
        });
    }
    for (int t = 0; t < writers; ++t) {
        threads.emplace_back([&] {
            for (;;) {
                int f;
                {
                    std::unique_lock<std::mutex> lk(P.mu);
                    P.cv.wait(lk, [&] { return P.abort || writers_done || qhead < write_queue.size(); });
                    if (P.abort) return;
                    if (qhead >= write_queue.size()) return;  // done and drained
                    f = write_queue[qhead++];
                }
                HostSet& s = P.sets[f % nsets];
                const auto a = clock::now();
                try {
                    const std::string stem = (fs::path(out_dir) / stem_of(frames[f].first)).string();
                    stereotk::RgbImage img(s.w, s.h);
                    std::memcpy(img.data.data(), s.out, img.data.size());
                    stereotk::save_rgb(img, stem + ext);
                    if (want_dense) {
                        stereotk::DisparityMap d(s.w, s.h);
                        std::memcpy(d.values.data(), s.dense, d.values.size() * 2);
                        stereotk::save_disparity(d, stem + "_disp.pgm", opts->disparity_scale);
                    }
                } catch (const std::exception& e) {
                    P.fail(classify(e), e.what());
                    return;
                }
                {
                    std::lock_guard<std::mutex> g(acc_mu);
                    write_s += std::chrono::duration<double>(clock::now() - a).count();
                }
                std::lock_guard<std::mutex> g(P.mu);
                s.state = HostSet::FREE;
                P.cv.notify_all();
            }
        });
    }

    // Main thread: submit in frame order, retire frame f - slots before its
    // GPU slot is reused.
    double gpu_wait_s = 0.0;
    auto retire = [&](int f) -> bool {
        HostSet& s = P.sets[f % nsets];
        const auto a = clock::now();
        stk_stats st{};
        const stk_status rc = stk_frame_wait(ctx, f % slots, &st, nullptr, nullptr);
        gpu_wait_s += std::chrono::duration<double>(clock::now() - a).count();
        if (rc != STK_OK) {
            P.fail(rc, stk_last_error(ctx));
            return false;
        }
        matched += st.matched;
        pixels += st.pixels;
        std::lock_guard<std::mutex> g(P.mu);
        s.state = HostSet::WRITING;
        write_queue.push_back(f);
        P.cv.notify_all();
        return true;
    };
    for (int f = 0; f < n && !P.abort; ++f) {
        if (f >= slots && !retire(f - slots)) break;
        HostSet& s = P.sets[f % nsets];
        {
            std::unique_lock<std::mutex> lk(P.mu);
            P.cv.wait(lk, [&] { return P.abort || (s.state == HostSet::DECODED && s.frame == f); });
            if (P.abort) break;
            s.state = HostSet::ON_GPU;
        }
        stk_frame_out o{};
        o.refocused = s.out;
        o.dense = s.dense;
        const stk_status rc = stk_frame_submit(ctx, f % slots, s.left, s.right, s.w, s.h, cfg, focus, &o, 0);
        if (rc != STK_OK) {
            P.fail(rc, stk_last_error(ctx));
            break;
        }
    }
    if (!P.abort)
        for (int f = std::max(0, n - slots); f < n; ++f)
            if (!retire(f)) break;
    {
        std::lock_guard<std::mutex> g(P.mu);
        writers_done = true;
        P.cv.notify_all();
    }
    if (P.abort) {  // drain anything still on the GPU before the buffers go away
        for (int s = 0; s < slots; ++s) stk_frame_wait(ctx, s, nullptr, nullptr, nullptr);
    }
    for (std::thread& t : threads) t.join();
    const double wall = std::chrono::duration<double>(clock::now() - t0).count();
    for (HostSet& s : P.sets) {
        stk_host_free(s.left);
        stk_host_free(s.right);
        stk_host_free(s.out);
        stk_host_free(s.dense);
    }
    if (report) {
        report->frames = P.abort ? 0 : n;
        report->frames_total = static_cast<int>(all.size());
        report->wall_s = wall;
        report->frames_per_s = wall > 0.0 && !P.abort ? n / wall : 0.0;
        report->decode_s = decode_s;
        report->write_s = write_s;
        report->gpu_wait_s = gpu_wait_s;
        report->matched_fraction = pixels ? double(matched) / double(pixels) : 0.0;
    }
    if (P.first_status != STK_OK) {
        stk::set_thread_error(P.first_error);
        return P.first_status;
    }
    return STK_OK;
}
