// stereotk_cli.cpp -- the reference's command-line front end
// (/root/reference/proj/tools/main.cpp) on the B200 library: the same four
// subcommands (depth, refocus, eval, bench), flags, JSON config precedence
// (flags > config file > defaults), stdout JSON shapes and exit codes
// (0 ok; 2 usage, parameter, format and I/O errors; 1 anything else), built
// as paper_2001_07809_b200/stereotk against libstk_b200.so (SURVEY.md §8f
// row 4).  Every pipeline stage runs on the GPU through the stereotk:: drop-in.
//
// The reference parses flags with CLI11 and JSON with nlohmann (vendored,
// absent here); this file carries a small option parser and a JSON reader of
// its own with the behaviour the reference's CLI tests pin
// (tests/test_cli.cpp): required flags and positionals, --name value and
// --name=value, conversion errors, unknown flags and keys -> exit 2.
#include <algorithm>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "stereotk/stereotk_b200.hpp"
#include "stk_b200.h"

namespace fs = std::filesystem;
using namespace stereotk;

namespace {

// ------------------------------------------------------------------- JSON --
struct Json {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    bool integral = false;
    std::string str;
    std::vector<Json> arr;
    std::map<std::string, Json> obj;  // nlohmann's default object is a sorted map

    const char* type_name() const {
        static const char* n[] = {"null", "boolean", "number", "string", "array", "object"};
        return n[kind];
    }
    // nlohmann get<int>() / get<double>(): numbers and booleans convert, the
    // rest is type_error 302.
    double number(const std::string& want) const {
        if (kind == Number) return num;
        if (kind == Bool) return b ? 1.0 : 0.0;
        throw std::runtime_error("[json.exception.type_error.302] type must be " + want + ", but is " +
                                 type_name());
    }
};

struct JsonParser {
    const std::string& s;
    std::size_t p = 0;

    [[noreturn]] void fail(const std::string& what) const {
        throw std::runtime_error("[json.exception.parse_error.101] parse error at byte " +
                                 std::to_string(p + 1) + ": " + what);
    }
    void ws() {
        while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\n' || s[p] == '\r')) ++p;
    }
    bool lit(const char* w) {
        const std::size_t n = std::strlen(w);
        if (s.compare(p, n, w) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    Json value() {
        ws();
        if (p >= s.size()) fail("unexpected end of input");
        Json j;
        const char c = s[p];
        if (c == '{') {
            j.kind = Json::Object;
            ++p;
            ws();
            if (p < s.size() && s[p] == '}') {
                ++p;
                return j;
            }
            for (;;) {
                ws();
                if (p >= s.size() || s[p] != '"') fail("expected object key");
                std::string k = string();
                ws();
                if (p >= s.size() || s[p] != ':') fail("expected ':'");
                ++p;
                j.obj[k] = value();
                ws();
                if (p < s.size() && s[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < s.size() && s[p] == '}') {
                    ++p;
                    return j;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            j.kind = Json::Array;
            ++p;
            ws();
            if (p < s.size() && s[p] == ']') {
                ++p;
                return j;
            }
            for (;;) {
                j.arr.push_back(value());
                ws();
                if (p < s.size() && s[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < s.size() && s[p] == ']') {
                    ++p;
                    return j;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            j.kind = Json::String;
            j.str = string();
            return j;
        }
        if (lit("true")) {
            j.kind = Json::Bool;
            j.b = true;
            return j;
        }
        if (lit("false")) {
            j.kind = Json::Bool;
            return j;
        }
        if (lit("null")) return j;
        // number: -?(0|[1-9][0-9]*)(\.[0-9]+)?([eE][+-]?[0-9]+)?
        const std::size_t st = p;
        if (s[p] == '-') ++p;
        auto digits = [&] {
            const std::size_t d = p;
            while (p < s.size() && std::isdigit(static_cast<unsigned char>(s[p]))) ++p;
            return p - d;
        };
        if (p < s.size() && s[p] == '0') {
            ++p;
        } else if (!digits()) {
            fail("invalid literal");
        }
        bool integral = true;
        if (p < s.size() && s[p] == '.') {
            ++p;
            integral = false;
            if (!digits()) fail("invalid number");
        }
        if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
            ++p;
            integral = false;
            if (p < s.size() && (s[p] == '+' || s[p] == '-')) ++p;
            if (!digits()) fail("invalid number");
        }
        j.kind = Json::Number;
        j.integral = integral;
        j.num = std::strtod(s.c_str() + st, nullptr);
        return j;
    }
    std::string string() {
        ++p;  // opening quote
        std::string out;
        while (p < s.size() && s[p] != '"') {
            char c = s[p++];
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                out += c;
                continue;
            }
            if (p >= s.size()) break;
            c = s[p++];
            switch (c) {
                case '"': out += '"'; break;
                case '\\': out += '\\'; break;
                case '/': out += '/'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'n': out += '\n'; break;
                case 'r': out += '\r'; break;
                case 't': out += '\t'; break;
                case 'u': {
                    if (p + 4 > s.size()) fail("bad \\u escape");
                    const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(p, 4), nullptr, 16));
                    p += 4;
                    if (cp < 0x80) {
                        out += static_cast<char>(cp);
                    } else if (cp < 0x800) {
                        out += static_cast<char>(0xC0 | (cp >> 6));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    } else {
                        out += static_cast<char>(0xE0 | (cp >> 12));
                        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    }
                    break;
                }
                default: fail("bad escape");
            }
        }
        if (p >= s.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Json document() {
        Json j = value();
        ws();
        if (p != s.size()) fail("trailing characters");
        return j;
    }
};

std::string json_string(const std::string& v) {
    std::string o = "\"";
    for (const char c : v) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", c);
                    o += b;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

// Compact JSON object with sorted keys (nlohmann::json::dump()).
struct JsonOut {
    std::map<std::string, std::string> fields;
    void num(const std::string& k, double v) { fields[k] = b200::json_number(v); }
    void integer(const std::string& k, long long v) { fields[k] = std::to_string(v); }
    void str(const std::string& k, const std::string& v) { fields[k] = json_string(v); }
    void obj(const std::string& k, const JsonOut& v) { fields[k] = v.dump(); }
    std::string dump() const {
        std::string o = "{";
        bool first = true;
        for (const auto& kv : fields) {
            if (!first) o += ",";
            first = false;
            o += json_string(kv.first) + ":" + kv.second;
        }
        return o + "}";
    }
};

// -------------------------------------------------------- option parsing --
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Option {
    std::string name;  // "--k" or a positional name
    std::string help;
    bool positional = false;
    bool required = false;
    std::function<void(const std::string&)> set;
    int count = 0;
};

struct Command {
    std::string name, help;
    std::vector<std::unique_ptr<Option>> opts;

    Option* add(const std::string& name, const std::string& help, std::function<void(const std::string&)> set,
                bool required = false) {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->help = help;
        o->positional = name.rfind("--", 0) != 0;
        o->required = required || o->positional;
        o->set = std::move(set);
        opts.push_back(std::move(o));
        return opts.back().get();
    }
    template <class T>
    Option* num(const std::string& name, T& dst, const std::string& help, bool required = false) {
        return add(
            name, help,
            [&dst, name](const std::string& v) {
                char* end = nullptr;
                errno = 0;
                if constexpr (std::is_integral_v<T>) {
                    const long x = std::strtol(v.c_str(), &end, 10);
                    if (v.empty() || *end || errno || x < INT32_MIN || x > INT32_MAX)
                        throw UsageError(name + ": Value " + v + " could not be converted");
                    dst = static_cast<T>(x);
                } else {
                    const double x = std::strtod(v.c_str(), &end);
                    if (v.empty() || *end || errno) throw UsageError(name + ": Value " + v + " could not be converted");
                    dst = x;
                }
            },
            required);
    }
    Option* text(const std::string& name, std::string& dst, const std::string& help, bool required = false) {
        return add(name, help, [&dst](const std::string& v) { dst = v; }, required);
    }

    std::string usage() const {
        std::ostringstream o;
        o << name << ": " << help << "\nUsage: stereotk " << name << " [OPTIONS]";
        for (const auto& op : opts)
            if (op->positional) o << " " << op->name;
        o << "\n\nOptions:\n  -h,--help                   Print this help message and exit\n";
        for (const auto& op : opts) {
            std::string n = op->positional ? op->name : op->name + " " + "VALUE";
            n.resize(std::max<std::size_t>(n.size() + 1, 28), ' ');
            o << "  " << n << op->help << (op->required ? " (REQUIRED)" : "") << "\n";
        }
        return o.str();
    }

    // Returns false when --help was printed.
    bool parse(const std::vector<std::string>& args) {
        std::vector<std::string> unexpected;
        std::size_t next_pos = 0;
        std::vector<Option*> pos;
        for (const auto& op : opts)
            if (op->positional) pos.push_back(op.get());
        for (std::size_t i = 0; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "-h" || a == "--help") {
                std::cout << usage();
                return false;
            }
            if (a.rfind("--", 0) == 0 && a.size() > 2) {
                std::string key = a, val;
                bool inline_val = false;
                const std::size_t eq = a.find('=');
                if (eq != std::string::npos) {
                    key = a.substr(0, eq);
                    val = a.substr(eq + 1);
                    inline_val = true;
                }
                Option* o = nullptr;
                for (const auto& op : opts)
                    if (!op->positional && op->name == key) o = op.get();
                if (!o) {
                    unexpected.push_back(a);
                    continue;
                }
                if (!inline_val) {
                    if (i + 1 >= args.size()) throw UsageError(key + ": 1 required VALUE missing");
                    val = args[++i];
                }
                o->set(val);
                ++o->count;
                continue;
            }
            if (next_pos < pos.size()) {
                pos[next_pos]->set(a);
                ++pos[next_pos]->count;
                ++next_pos;
            } else {
                unexpected.push_back(a);
            }
        }
        if (!unexpected.empty()) {
            std::string m = "The following arguments were not expected:";
            for (const auto& u : unexpected) m += " " + u;
            throw UsageError(m);
        }
        for (const auto& op : opts)
            if (op->required && op->count == 0) throw UsageError(op->name + " is required");
        return true;
    }
};

// ------------------------------------------------ config file (main.cpp) --
struct ConfigBinding {
    const char* key;
    Option* option;
    std::function<void(const Json&)> apply;
};

// main.cpp:38-72: flags > config file > defaults.
void apply_config_file(const std::string& path, const std::vector<ConfigBinding>& bindings) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open config " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    Json doc;
    try {
        JsonParser jp{text};
        doc = jp.document();
    } catch (const std::runtime_error& e) {
        throw FormatError(path + ": " + e.what());
    }
    if (doc.kind != Json::Object) throw FormatError(path + ": config must be a JSON object");
    for (const auto& [key, value] : doc.obj) {
        const ConfigBinding* b = nullptr;
        for (const ConfigBinding& c : bindings)
            if (key == c.key) b = &c;
        if (!b) throw ParamError("config " + path + ": unknown key '" + key + "'");
        if (b->option->count > 0) continue;
        try {
            b->apply(value);
        } catch (const std::runtime_error& e) {
            throw FormatError(path + ": key '" + key + "': " + e.what());
        }
    }
}

struct PipelineFlags {
    PipelineConfig config;
    std::string config_path;
    Option *k = nullptr, *window = nullptr, *max_disparity = nullptr, *threshold = nullptr,
           *prune_fraction = nullptr, *workers = nullptr;

    void add(Command& c, bool with_workers = true) {
        k = c.num("--k", config.k, "Lightness clusters");
        window = c.num("--window", config.window, "SAD window side (odd)");
        max_disparity = c.num("--max-disparity", config.max_disparity, "Largest disparity searched");
        threshold = c.num("--threshold", config.threshold, "Column-pass discontinuity threshold");
        prune_fraction = c.num("--prune-fraction", config.prune_fraction, "Boundary noise budget in [0, 1)");
        workers = c.num(with_workers ? "--workers" : "--pipeline-workers", config.workers,
                        "Threads for the parallel kernels (validated; the GPU result is identical)");
        c.text("--config", config_path, "JSON config file (flags win)");
    }
    std::vector<ConfigBinding> bindings() {
        auto as_int = [](const Json& v) { return static_cast<int>(v.number("number")); };
        return {
            {"k", k, [this, as_int](const Json& v) { config.k = as_int(v); }},
            {"window", window, [this, as_int](const Json& v) { config.window = as_int(v); }},
            {"max_disparity", max_disparity, [this, as_int](const Json& v) { config.max_disparity = as_int(v); }},
            {"threshold", threshold, [this, as_int](const Json& v) { config.threshold = as_int(v); }},
            {"prune_fraction", prune_fraction,
             [this](const Json& v) { config.prune_fraction = v.number("number"); }},
            {"workers", workers, [this, as_int](const Json& v) { config.workers = as_int(v); }},
        };
    }
};

// ------------------------------------------------------------ subcommands --
GrayImage mask_to_gray(const BoundaryMask& m) {
    GrayImage g(m.width, m.height);
    for (std::size_t i = 0; i < g.data.size(); ++i) g.data[i] = m.mask[i] ? 255 : 0;
    return g;
}

// main.cpp:131-158
void dump_depth_debug(const DepthResult& r, double scale, const std::string& dir) {
    fs::create_directories(dir);
    save_gray(r.left_lightness, dir + "/lightness_left.pgm");
    save_gray(r.right_lightness, dir + "/lightness_right.pgm");
    GrayImage labels(r.labels.width, r.labels.height);
    const int k = r.clustering.k();
    for (std::size_t i = 0; i < labels.data.size(); ++i)
        labels.data[i] = static_cast<std::uint8_t>(k > 1 ? std::lround(r.labels.labels[i] * 255.0 / (k - 1)) : 0);
    save_gray(labels, dir + "/labels.pgm");
    save_gray(mask_to_gray(r.boundary_raw), dir + "/boundary_raw.pgm");
    save_gray(mask_to_gray(r.boundary_refined), dir + "/boundary_refined.pgm");
    save_gray(mask_to_gray(r.boundary_anchored), dir + "/boundary_anchored.pgm");
    save_disparity(r.sparse, dir + "/sparse.pgm", scale);
    save_disparity(r.row_filled, dir + "/row_filled.pgm", scale);
    save_disparity(r.dense, dir + "/dense.pgm", scale);
}

// main.cpp:160-180
std::string stats_json(const DepthResult& r, const StageTimes& t) {
    JsonOut o, st;
    o.integer("width", r.dense.width);
    o.integer("height", r.dense.height);
    o.integer("boundary_raw", static_cast<long long>(r.stats.boundary_raw));
    o.integer("boundary_refined", static_cast<long long>(r.stats.boundary_refined));
    o.integer("matched", static_cast<long long>(r.stats.matched));
    o.num("matched_fraction", r.stats.matched_fraction);
    o.num("known_fraction", r.stats.known_fraction);
    o.integer("iterations", r.clustering.iterations_run);
    st.num("convert", t.convert);
    st.num("segment", t.segment);
    st.num("boundary", t.boundary);
    st.num("match", t.match);
    st.num("fill", t.fill);
    st.num("peek", t.peek);
    st.num("total", t.total());
    o.obj("times_ms", st);
    return o.dump();
}

// main.cpp:183-218
std::vector<std::pair<int, int>> parse_focus(const std::string& text) {
    std::vector<std::pair<int, int>> ranges;
    std::stringstream in(text);
    std::string part;
    while (std::getline(in, part, ',')) {
        const std::size_t colon = part.find(':');
        if (colon == std::string::npos) throw ParamError("focus range '" + part + "' is not of the form lo:hi");
        int lo = 0, hi = 0;
        try {
            std::size_t used = 0;
            lo = std::stoi(part.substr(0, colon), &used);
            if (used != colon) throw std::invalid_argument(part);
            const std::string rest = part.substr(colon + 1);
            hi = std::stoi(rest, &used);
            if (used != rest.size()) throw std::invalid_argument(part);
        } catch (const std::exception&) {
            throw ParamError("focus range '" + part + "' is not of the form lo:hi");
        }
        if (lo < 0 || lo > hi) throw ParamError("focus range '" + part + "' is empty or negative");
        ranges.emplace_back(lo, hi);
    }
    if (ranges.empty()) throw ParamError("no focus ranges given");
    return ranges;
}

// main.cpp:220-241
std::vector<int> parse_worker_list(const std::string& text) {
    std::vector<int> w;
    std::stringstream in(text);
    std::string part;
    while (std::getline(in, part, ',')) {
        try {
            std::size_t used = 0;
            const int v = std::stoi(part, &used);
            if (used != part.size()) throw std::invalid_argument(part);
            w.push_back(v);
        } catch (const std::exception&) {
            throw ParamError("worker list entry '" + part + "' is not an integer");
        }
    }
    if (w.empty()) throw ParamError("empty worker list");
    return w;
}

struct DepthOpts {
    std::string left, right, out, debug_dir;
    double scale = 8.0;
    PipelineFlags pipeline;
    Option* scale_opt = nullptr;
};

int run_depth(DepthOpts& o) {  // main.cpp:294-316
    if (!o.pipeline.config_path.empty()) {
        auto b = o.pipeline.bindings();
        b.push_back({"scale", o.scale_opt, [&](const Json& v) { o.scale = v.number("number"); }});
        apply_config_file(o.pipeline.config_path, b);
    }
    if (!(o.scale > 0.0)) throw ParamError("scale must be positive, got " + std::to_string(o.scale));
    const RgbImage left = load_image(o.left);
    const RgbImage right = load_image(o.right);
    StageTimes times;
    const DepthResult r = run_depth_pipeline(left, right, o.pipeline.config, &times);
    save_disparity(r.dense, o.out, o.scale);
    if (!o.debug_dir.empty()) dump_depth_debug(r, o.scale, o.debug_dir);
    std::cout << stats_json(r, times) << "\n";
    return 0;
}

struct RefocusOpts {
    std::string left, right, out, focus_text, debug_dir;
    double sigma = 2.0;
    int kernel_size = 0;
    PipelineFlags pipeline;
    Option *sigma_opt = nullptr, *kernel_opt = nullptr;
};

int run_refocus(RefocusOpts& o) {  // main.cpp:327-379
    if (!o.pipeline.config_path.empty()) {
        auto b = o.pipeline.bindings();
        b.push_back({"sigma", o.sigma_opt, [&](const Json& v) { o.sigma = v.number("number"); }});
        b.push_back({"kernel_size", o.kernel_opt,
                     [&](const Json& v) { o.kernel_size = static_cast<int>(v.number("number")); }});
        apply_config_file(o.pipeline.config_path, b);
    }
    if (!(o.sigma > 0.0)) throw ParamError("sigma must be positive, got " + std::to_string(o.sigma));
    if (o.kernel_size != 0 && (o.kernel_size < 1 || o.kernel_size % 2 == 0))
        throw ParamError("kernel size must be odd and positive, got " + std::to_string(o.kernel_size));
    FocusSpec focus;
    focus.sigma = o.sigma;
    focus.ranges = parse_focus(o.focus_text);
    for (auto& [lo, hi] : focus.ranges) {  // ranges past the search range are trimmed to it
        lo = std::min(lo, o.pipeline.config.max_disparity);
        hi = std::min(hi, o.pipeline.config.max_disparity);
    }
    const RgbImage left = load_image(o.left);
    const RgbImage right = load_image(o.right);
    DepthResult depth;
    const RgbImage out = run_refocus_pipeline(left, right, o.pipeline.config, focus, o.kernel_size, &depth);
    save_rgb(out, o.out);
    if (!o.debug_dir.empty()) {
        dump_depth_debug(depth, 8.0, o.debug_dir);
        GrayImage visible = build_blur_map(depth.dense, focus, o.pipeline.config.max_disparity);
        for (std::uint8_t& v : visible.data) v = v ? 255 : 0;
        save_gray(visible, o.debug_dir + "/blur_map.pgm");
    }
    JsonOut j;
    j.str("out", o.out);
    j.num("matched_fraction", depth.stats.matched_fraction);
    std::cout << j.dump() << "\n";
    return 0;
}

struct EvalOpts {
    std::string computed, truth;
    double scale = 0.0, delta = 1.0;
    int workers = 1;
};

int run_eval(const EvalOpts& o) {  // main.cpp:388-405
    if (!(o.scale > 0.0)) throw ParamError("scale must be positive, got " + std::to_string(o.scale));
    if (o.delta < 0.0) throw ParamError("delta must be >= 0, got " + std::to_string(o.delta));
    const DisparityMap computed = load_disparity(o.computed, o.scale);
    const DisparityMap truth = load_ground_truth(o.truth, o.scale);
    std::cout << eval_report_json(bad_pixel_rate(computed, truth, o.delta, o.workers)) << "\n";
    return 0;
}

struct BenchOpts {
    std::string frames_dir, workers_text = "1,4", csv_path, gpus_text, focus_text;
    double sigma = 2.0;
    int kernel_size = 0;
    PipelineFlags pipeline;
};

// --gpus (B200 extension): the batch per GPU count,
// frame f -> GPU f mod G; CSV with a blur row and GB/s columns; the summary
// adds frames/s per count.
int run_bench_gpus(BenchOpts& o) {
    std::vector<int> gpus;
    try {
        gpus = parse_worker_list(o.gpus_text);
    } catch (const ParamError&) {
        throw ParamError("GPU list '" + o.gpus_text + "' is not a comma-separated list of integers");
    }
    const std::vector<StereoPair> frames = load_frames(o.frames_dir);
    FocusSpec focus;
    focus.sigma = o.sigma;
    if (!o.focus_text.empty()) {
        focus.ranges = parse_focus(o.focus_text);
        for (auto& [lo, hi] : focus.ranges) {
            lo = std::min(lo, o.pipeline.config.max_disparity);
            hi = std::min(hi, o.pipeline.config.max_disparity);
        }
    }
    const std::vector<GpuBenchReport> reports = run_benchmark_gpus(
        frames, gpus, o.pipeline.config, o.focus_text.empty() ? nullptr : &focus, o.kernel_size);
    const std::string csv = benchmark_csv(reports);
    if (o.csv_path.empty()) {
        std::cout << csv;
        return 0;
    }
    std::ofstream out(o.csv_path, std::ios::trunc);
    if (!out) throw IoError("cannot open " + o.csv_path + " for writing");
    out << csv;
    if (!out) throw IoError("write failed: " + o.csv_path);
    JsonOut summary, speedup, fps;
    summary.str("csv", o.csv_path);
    summary.integer("frames", reports.front().frames);
    for (const GpuBenchReport& r : reports) {
        speedup.num(std::to_string(r.gpus), r.speedup);
        fps.num(std::to_string(r.gpus), r.frames_per_s);
    }
    summary.obj("frames_per_s", fps);
    summary.obj("speedup", speedup);
    std::cout << summary.dump() << "\n";
    return 0;
}

int run_bench(BenchOpts& o) {  // main.cpp:412-440
    if (!o.pipeline.config_path.empty()) apply_config_file(o.pipeline.config_path, o.pipeline.bindings());
    if (!o.gpus_text.empty()) return run_bench_gpus(o);
    const std::vector<int> workers = parse_worker_list(o.workers_text);
    const std::vector<StereoPair> frames = load_frames(o.frames_dir);
    const std::vector<BenchReport> reports = run_benchmark(frames, workers, o.pipeline.config);
    const std::string csv = benchmark_csv(reports);
    if (o.csv_path.empty()) {
        std::cout << csv;
        return 0;
    }
    std::ofstream out(o.csv_path, std::ios::trunc);
    if (!out) throw IoError("cannot open " + o.csv_path + " for writing");
    out << csv;
    if (!out) throw IoError("write failed: " + o.csv_path);
    JsonOut summary, speedup;
    summary.str("csv", o.csv_path);
    summary.integer("frames", reports.front().frames);
    for (const BenchReport& r : reports) speedup.num(std::to_string(r.workers), r.speedup);
    summary.obj("speedup", speedup);
    std::cout << summary.dump() << "\n";
    return 0;
}

// B200 extension (no reference counterpart): a directory of frame pairs
// refocused with file decode, PCIe copies, kernels and encode overlapped
// (stk_video_refocus), optionally one shard of the frames per GPU.
struct VideoOpts {
    std::string in_dir, out_dir, focus_text;
    double sigma = 2.0, disparity_scale = 0.0;
    int kernel_size = 0, slots = 3, decode_threads = 4, write_threads = 2, device = -1;
    int shard_index = 0, shard_count = 1;
    std::string png = "0";
    PipelineFlags pipeline;
};

int run_video(VideoOpts& o) {
    if (!o.pipeline.config_path.empty()) apply_config_file(o.pipeline.config_path, o.pipeline.bindings());
    if (!(o.sigma > 0.0)) throw ParamError("sigma must be positive, got " + std::to_string(o.sigma));
    if (o.kernel_size != 0 && (o.kernel_size < 1 || o.kernel_size % 2 == 0))
        throw ParamError("kernel size must be odd and positive, got " + std::to_string(o.kernel_size));
    if (o.slots < 1) throw ParamError("slots must be >= 1, got " + std::to_string(o.slots));
    auto ranges = parse_focus(o.focus_text);
    std::vector<int> lo, hi;
    for (auto& [a, b] : ranges) {
        lo.push_back(std::min(a, o.pipeline.config.max_disparity));
        hi.push_back(std::min(b, o.pipeline.config.max_disparity));
    }
    const PipelineConfig& c = o.pipeline.config;
    const stk_config cfg{c.k, c.window, c.max_disparity, c.threshold, c.prune_fraction, c.workers};
    const stk_focus fo{lo.data(), hi.data(), static_cast<int>(lo.size()), o.sigma, o.kernel_size,
                       b200::fast_blur() ? 0 : 1};
    const stk_video_opts vo{o.slots, o.decode_threads, o.write_threads, o.png == "1" || o.png == "true",
                            o.disparity_scale, o.shard_index, o.shard_count};
    int device = o.device;
    if (device < 0) {
        const char* e = std::getenv("STK_DEVICE");
        device = e ? std::atoi(e) : 0;
    }
    auto check = [](stk_status s, const stk_ctx* ctx) {
        if (s == STK_OK) return;
        const std::string m = stk_last_error(ctx);
        if (s == STK_EPARAM) throw ParamError(m);
        if (s == STK_EIO) throw IoError(m);
        if (s == STK_EFORMAT) throw FormatError(m);
        throw std::runtime_error(m);
    };
    check(stk_validate_config(&cfg), nullptr);
    stk_ctx* ctx = nullptr;
    check(stk_create(device, 0, 0, o.slots, &ctx), nullptr);
    stk_video_report rep{};
    const stk_status st = stk_video_refocus(ctx, o.in_dir.c_str(), o.out_dir.c_str(), &cfg, &fo, &vo, &rep);
    stk_destroy(ctx);
    check(st, nullptr);
    JsonOut j;
    j.integer("frames", rep.frames);
    j.integer("frames_total", rep.frames_total);
    j.num("wall_s", rep.wall_s);
    j.num("frames_per_s", rep.frames_per_s);
    j.num("decode_s", rep.decode_s);
    j.num("write_s", rep.write_s);
    j.num("gpu_wait_s", rep.gpu_wait_s);
    j.num("matched_fraction", rep.matched_fraction);
    j.str("out_dir", o.out_dir);
    std::cout << j.dump() << "\n";
    return 0;
}

const char* kAppHelp =
    "Boundary-driven stereo depth estimation and selective refocus (B200)\n"
    "Usage: stereotk [OPTIONS] SUBCOMMAND\n\n"
    "Options:\n  -h,--help                   Print this help message and exit\n\n"
    "Subcommands:\n"
    "  depth                       Estimate a dense disparity map from a rectified pair\n"
    "  refocus                     Blur everything outside the in-focus disparity ranges\n"
    "  eval                        Compare a computed disparity map against ground truth\n"
    "  bench                       Time the pipeline serial vs parallel over a frame batch\n"
    "  video                       Refocus a directory of frame pairs, decode/GPU/encode overlapped\n";

}  // namespace

int main(int argc, char** argv) {
    DepthOpts depth_opts;
    Command depth{"depth", "Estimate a dense disparity map from a rectified pair", {}};
    depth.text("--left", depth_opts.left, "Left image (PNG/PPM)", true);
    depth.text("--right", depth_opts.right, "Right image (PNG/PPM)", true);
    depth.text("--out", depth_opts.out, "Output disparity PGM", true);
    depth_opts.scale_opt = depth.num("--scale", depth_opts.scale, "Output encoding scale (value = d * scale)");
    depth.text("--debug-dir", depth_opts.debug_dir, "Dump per-stage images into this directory");
    depth_opts.pipeline.add(depth);

    RefocusOpts refocus_opts;
    Command refocus{"refocus", "Blur everything outside the in-focus disparity ranges", {}};
    refocus.text("--left", refocus_opts.left, "Left image (PNG/PPM)", true);
    refocus.text("--right", refocus_opts.right, "Right image (PNG/PPM)", true);
    refocus.text("--out", refocus_opts.out, "Output image (PNG/PPM)", true);
    refocus.text("--focus", refocus_opts.focus_text, "In-focus disparity ranges lo:hi[,lo:hi...]", true);
    refocus_opts.sigma_opt = refocus.num("--sigma", refocus_opts.sigma, "Gaussian blur strength");
    refocus_opts.kernel_opt =
        refocus.num("--kernel-size", refocus_opts.kernel_size, "Odd kernel side (default: derived from sigma)");
    refocus.text("--debug-dir", refocus_opts.debug_dir, "Dump per-stage images into this directory");
    refocus_opts.pipeline.add(refocus);

    EvalOpts eval_opts;
    Command eval{"eval", "Compare a computed disparity map against ground truth", {}};
    eval.text("computed", eval_opts.computed, "Computed disparity PGM");
    eval.text("--truth", eval_opts.truth, "Ground-truth image", true);
    eval.num("--scale", eval_opts.scale, "Ground-truth encoding scale (value = d * scale)", true);
    eval.num("--delta", eval_opts.delta, "Bad-pixel tolerance");
    eval.num("--workers", eval_opts.workers, "Comparison threads (validated; GPU reduction)");

    BenchOpts bench_opts;
    Command bench{"bench", "Time the pipeline serial vs parallel over a frame batch", {}};
    bench.text("frames", bench_opts.frames_dir, "Directory of <stem>_L/<stem>_R frame pairs");
    bench.text("--workers", bench_opts.workers_text, "Comma-separated worker counts (must include 1)");
    bench.text("--csv", bench_opts.csv_path, "Write the CSV here instead of stdout");
    bench.text("--gpus", bench_opts.gpus_text,
               "B200: comma-separated GPU counts (must include 1); frame f -> GPU f mod G");
    bench.text("--focus", bench_opts.focus_text, "B200 --gpus: in-focus ranges lo:hi[,...] (adds the blur)");
    bench.num("--sigma", bench_opts.sigma, "B200 --gpus: Gaussian blur strength");
    bench.num("--kernel-size", bench_opts.kernel_size, "B200 --gpus: odd kernel side (default from sigma)");
    bench_opts.pipeline.add(bench, /*with_workers=*/false);

    VideoOpts video_opts;
    Command video{"video", "Refocus a directory of <stem>_L/_R frame pairs (B200 extension)", {}};
    video.text("frames", video_opts.in_dir, "Directory of <stem>_L/<stem>_R frame pairs");
    video.text("--out-dir", video_opts.out_dir, "Output directory (<stem>.ppm|.png)", true);
    video.text("--focus", video_opts.focus_text, "In-focus disparity ranges lo:hi[,lo:hi...]", true);
    video.num("--sigma", video_opts.sigma, "Gaussian blur strength");
    video.num("--kernel-size", video_opts.kernel_size, "Odd kernel side (default: derived from sigma)");
    video.text("--png", video_opts.png, "1: write PNG instead of PPM");
    video.num("--disparity-scale", video_opts.disparity_scale, "> 0: also write <stem>_disp.pgm at this scale");
    video.num("--slots", video_opts.slots, "GPU frames in flight");
    video.num("--decode-threads", video_opts.decode_threads, "Host decoder threads");
    video.num("--write-threads", video_opts.write_threads, "Host encoder threads");
    video.num("--device", video_opts.device, "CUDA device (default $STK_DEVICE or 0)");
    video.num("--shard-index", video_opts.shard_index, "Process frames f with f % shard-count == shard-index");
    video.num("--shard-count", video_opts.shard_count, "Number of shards (one per GPU)");
    video_opts.pipeline.add(video);

    Command* cmds[] = {&depth, &refocus, &eval, &bench, &video};
    std::vector<std::string> args(argv + 1, argv + argc);
    Command* chosen = nullptr;
    try {
        std::size_t i = 0;
        for (; i < args.size(); ++i) {
            if (args[i] == "-h" || args[i] == "--help") {
                std::cout << kAppHelp;
                return 0;
            }
            for (Command* c : cmds)
                if (args[i] == c->name) chosen = c;
            if (chosen) break;
            throw UsageError("The following argument was not expected: " + args[i]);
        }
        if (!chosen) throw UsageError("A subcommand is required");
        if (!chosen->parse(std::vector<std::string>(args.begin() + i + 1, args.end()))) return 0;
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 2;
    }

    try {
        if (chosen == &depth) return run_depth(depth_opts);
        if (chosen == &refocus) return run_refocus(refocus_opts);
        if (chosen == &eval) return run_eval(eval_opts);
        if (chosen == &bench) return run_bench(bench_opts);
        if (chosen == &video) return run_video(video_opts);
    } catch (const ParamError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const FormatError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
