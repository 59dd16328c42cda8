// stk_capi.cu -- the C-ABI (include/stk_b200.h): context, per-slot HBM
// planes, TMA descriptors, frame enqueue (optionally as a CUDA graph), and the
// synchronous per-stage entries used as the parity surface.
//
// Validation mirrors the reference's checks and message text so the C++ shim
// can rethrow stereotk::ParamError verbatim (pipeline.cpp:23-60,
// segmentation.cpp:64-93, boundary.cpp:150-185, stereo.cpp:32-58,
// reconstruct.cpp:50-55, refocus.cpp:16-57).
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <nvtx3/nvToolsExtCudaRt.h>

#include "stk_b200.h"
#include "stk_internal.cuh"

using namespace stk;

struct stk_ctx;

namespace {

thread_local std::string t_err;

// Disparities are int16 (DisparityMap, stereo.hpp:13-40), so no map holds a
// value above 32767: the focus LUT never needs more entries than this.
constexpr int kMaxLut = 32768;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct TMap {
    CUtensorMap map;
    const void* ptr = nullptr;
    int W = -1, H = -1, pitch = -1, bw = -1, bh = -1, esz = -1;
};

// Everything a captured frame graph bakes in: geometry, configuration and
// every device pointer its nodes read or write (the caller's buffers and the
// slot's focus tables, which upload_focus may reallocate).  Zeroed as a
// whole (padding included) so memcmp is a field-by-field comparison.
struct GraphKey {
    int W, H, kcfg, window, D, thr, full, focus, hw, exact, lut_len, sad, want_raw, pad_;
    double frac;
    const void *rgbL, *rgbR, *out_rgb, *dense, *lut, *g1, *g2, *blur_tmp;
    GraphKey() { std::memset(this, 0, sizeof(*this)); W = H = -1; }
    bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};

struct Slot {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[8] = {};
    cudaEvent_t done = nullptr;
    char* base = nullptr;
    size_t bytes = 0;
    // layout for the current frame geometry
    int W = 0, H = 0, P = 0;
    int sms = 148;  // copied from the context at creation
    uint8_t *rgbL, *rgbR, *grayL, *grayR, *mraw, *mref, *mprn, *manc, *out_rgb;
    uint16_t *labels16, *scratch16;
    uint32_t* mbits;
    int32_t *par, *rank, *roots;
    uint32_t *cnt, *szhist, *list, *tile_off;
    unsigned long long* lb;
    int lb_stride = 0;
    int16_t *sparse, *rowf, *dense;
    uint32_t *rbits, *sbits;  // refined bits, size-s* root bitmap (k_bnd.cu)
    int32_t *runroot, *bord;  // per-run component root, tile border roots
    int sbits_words = 0;
    DevScalars* sc = nullptr;
    DevScalars* h_sc = nullptr;  // pinned mirror
    // focus tables
    uint8_t* d_lut = nullptr;
    int lut_cap = 0;
    float* d_g1 = nullptr;
    double* d_g2 = nullptr;
    int g_cap = 0;
    std::vector<uint8_t> h_lut;
    std::vector<float> h_g1;
    std::vector<double> h_g2;
    // pinned staging of the focus tables: uploads are stream-ordered async
    // copies (no host synchronisation when the focus changes between frames)
    uint8_t* p_lut = nullptr;
    float* p_g1 = nullptr;
    double* p_g2 = nullptr;
    // vertical-sum plane of the global-memory blur fallback (very wide kernels)
    float* blur_tmp = nullptr;
    size_t blur_tmp_bytes = 0;
    // label_components scratch
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    // tensor maps
    TMap tm_sadL, tm_sadR;
    // graph
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey;
    // pending frame
    bool pending = false;
    bool timed = false;
    bool graph = false;
    bool captured = false;
    int kernels = 0;
    int k_for_out = 0;
    Frame f{};
    stk_frame_out out{};
};

}  // namespace

struct stk_ctx {
    int device = 0;
    std::string err;
    LstarTables* d_tab = nullptr;
    uint8_t* d_lut = nullptr;  // exact 2^24-entry L* table (frame path), null = K1 arithmetic path
    std::vector<Slot> slots;
    int sad_kernel = SAD_AUTO;
    int use_graphs = 1;
    int sms = 148;  // cudaDevAttrMultiProcessorCount of `device` (grid sizing)
    EncodeTiledFn encode = nullptr;
};

namespace {

stk_status fail(stk_ctx* ctx, stk_status s, const std::string& msg) {
    t_err = msg;
    if (ctx) ctx->err = msg;
    return s;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, STK_ECUDA, std::string("cuda: ") + #call + ": " +            \
                                            cudaGetErrorString(e_));                      \
    } while (0)

std::string dims(int w, int h) { return std::to_string(w) + "x" + std::to_string(h); }

// ------------------------------------------------ L* tables (host libm) ---
// lightness.cpp:14-21, 44-49 evaluated with the same libm as the reference.
double srgb_to_linear(int v) {
    const double c = v / 255.0;
    return c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4);
}

int lstar_byte(double y) {
    const double eps = 216.0 / 24389.0, kappa = 24389.0 / 27.0;
    const double f = y > eps ? std::cbrt(y) : (kappa * y + 16.0) / 116.0;
    const double lstar = 116.0 * f - 16.0;
    long s = std::lround(lstar * 255.0 / 100.0);
    return (int)(s < 0 ? 0 : (s > 255 ? 255 : s));
}

void make_lstar_tables(LstarTables* t) {
    for (int v = 0; v < 256; ++v) t->linear[v] = srgb_to_linear(v);
    for (int v = 0; v < 256; ++v) {
        volatile double l = t->linear[v];  // plain IEEE products, no contraction
        t->prod[0][v] = 0.2126 * l;
        t->prod[1][v] = 0.7152 * l;
        t->prod[2][v] = 0.0722 * l;
        for (int c = 0; c < 3; ++c) t->fprod[c][v] = (float)t->prod[c][v];
    }
    t->thr[0] = -1.0;
    uint64_t hi_bits;
    const double two = 2.0;
    std::memcpy(&hi_bits, &two, 8);
    for (int v = 1; v < 256; ++v) {
        // smallest non-negative double y with L*(y) >= v, by bisection over the
        // IEEE-754 bit patterns (monotone for y >= 0)
        uint64_t lo = 0, hi = hi_bits;
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            double y;
            std::memcpy(&y, &mid, 8);
            if (lstar_byte(y) >= v) hi = mid;
            else lo = mid;
        }
        std::memcpy(&t->thr[v], &hi, 8);
    }
    // bucketed lookup: base[b] = #{v >= 1 : thr[v] <= b/NB}, tb[b] = the one
    // threshold strictly inside (b/NB, (b+1)/NB), or +inf
    const double NB = kLstarBuckets;
    int v = 1;
    for (int b = 0; b <= kLstarBuckets; ++b) {
        const double lo = b / NB, hi = (b + 1) / NB;
        while (v < 256 && t->thr[v] <= lo) ++v;
        t->base[b] = (unsigned char)(v - 1);
        t->tb[b] = (v < 256 && t->thr[v] < hi) ? t->thr[v] : INFINITY;
        if (v + 1 < 256 && t->thr[v + 1] < hi && t->thr[v] < hi) t->tb[b] = -INFINITY;  // flagged
        uint32_t q = 0xffffffu;
        if (std::isfinite(t->tb[b])) q = (uint32_t)((t->tb[b] * NB - b) * 16777216.0);  // exact, < 2^24
        t->bw[b] = (uint32_t)t->base[b] << 24 | q;
    }
    // K1's FP32 screen (k_lightness.cu): a screened Y' is within 5 * 2^-24 of
    // the reference's Y, so with a 2^-20 margin a sub-bucket without a
    // threshold in its widened span has one gray value for every pixel
    // screened into it
    const double E = std::ldexp(1.0, -20);
    int c = 0;  // thresholds <= lo
    for (int s = 0; s < 65536; ++s) {
        const double lo = s * std::ldexp(1.0, -16) - E, hi = (s + 1) * std::ldexp(1.0, -16) + E;
        while (c < 255 && t->thr[c + 1] <= lo) ++c;
        const bool inside = c < 255 && t->thr[c + 1] <= hi;
        t->sub[s] = inside || c >= 255 ? 0xffu : (uint8_t)c;
    }
    const double b255 = (t->thr[255] + E) * 8388608.0;  // 2^23: Y' mantissa units
    t->bright = 0x3f800000u | (uint32_t)std::ceil(b255);
}

bool lstar_buckets_ok(const LstarTables* t) {
    for (int b = 0; b <= kLstarBuckets; ++b)
        if (t->tb[b] == -INFINITY) return false;
    return true;
}

// --------------------------------------------------------------- layout ---
struct Layout {
    size_t off[32];
    size_t total;
};

enum {
    L_RGBL, L_RGBR, L_OUT, L_GRAYL, L_GRAYR, L_MRAW, L_MREF, L_MPRN, L_MANC, L_LAB16, L_SCR16,
    L_MBITS, L_PAR, L_CNT, L_RANK, L_SZH, L_ROOTS, L_LIST, L_TOFF, L_LB, L_SPARSE, L_ROWF,
    L_DENSE, L_SC, L_RBITS, L_RUNR, L_BORD, L_SBITS, L_COUNT
};

Layout layout_for(int W, int H, int* P_out, int* lb_stride_out) {
    const size_t N = (size_t)W * H;
    const int P = (int)align_up((size_t)std::max(W, 1), 64);
    const size_t PH = (size_t)P * H;
    const int TX = (W + kRowTile - 1) / kRowTile;
    const size_t n_tiles = (size_t)H * TX;
    const size_t n_chunks = (n_tiles + kTilesPerChunk - 1) / kTilesPerChunk;
    const int lb_stride = (int)n_chunks + 1;
    size_t sz[L_COUNT];
    sz[L_RGBL] = sz[L_RGBR] = sz[L_OUT] = 3 * N + 64;
    sz[L_GRAYL] = sz[L_GRAYR] = sz[L_MRAW] = sz[L_MREF] = sz[L_MPRN] = sz[L_MANC] = PH + 64;
    sz[L_LAB16] = 2 * N + 64;
    sz[L_SCR16] = 2 * PH + 64;
    sz[L_MBITS] = (size_t)H * TX * 4 * 4 + 64;
    sz[L_PAR] = sz[L_CNT] = sz[L_RANK] = sz[L_ROOTS] = sz[L_LIST] = 4 * N + 64;
    sz[L_SZH] = 4 * (N + 2) + 64;
    sz[L_TOFF] = 4 * (n_tiles + 1) + 64;
    sz[L_LB] = 8 * (size_t)LB_COUNT * lb_stride + 64;
    sz[L_SPARSE] = sz[L_ROWF] = sz[L_DENSE] = 2 * N + 64;
    sz[L_SC] = sizeof(DevScalars);
    // bit-packed boundary stage (k_bnd.cu)
    const size_t ctiles = (size_t)((W + 31) / 32) * ((H + 31) / 32);
    sz[L_RBITS] = sz[L_SBITS] = (size_t)H * TX * 4 * 4 + 64;
    sz[L_RUNR] = ctiles * 512 * 4 + 64;
    sz[L_BORD] = bord_bytes(W, H) + 64;  // region border labels (was sized per tile: short for tiny frames)
    Layout L;
    size_t o = 0;
    for (int i = 0; i < L_COUNT; ++i) {
        L.off[i] = o;
        o = align_up(o + sz[i], 256);
    }
    L.total = o;
    *P_out = P;
    *lb_stride_out = lb_stride;
    return L;
}

stk_status ensure_slot(stk_ctx* ctx, Slot& s, int W, int H) {
    if (s.W == W && s.H == H && s.base) return STK_OK;
    int P, lbs;
    const Layout L = layout_for(W, H, &P, &lbs);
    if (L.total > s.bytes) {
        if (s.base) {
            CK(cudaStreamSynchronize(s.st));
            CK(cudaFree(s.base));
            s.base = nullptr;
        }
        CK(cudaMalloc(&s.base, L.total));
        s.bytes = L.total;
    }
    char* b = s.base;
    s.W = W;
    s.H = H;
    s.P = P;
    s.lb_stride = lbs;
    s.rgbL = (uint8_t*)(b + L.off[L_RGBL]);
    s.rgbR = (uint8_t*)(b + L.off[L_RGBR]);
    s.out_rgb = (uint8_t*)(b + L.off[L_OUT]);
    s.grayL = (uint8_t*)(b + L.off[L_GRAYL]);
    s.grayR = (uint8_t*)(b + L.off[L_GRAYR]);
    s.mraw = (uint8_t*)(b + L.off[L_MRAW]);
    s.mref = (uint8_t*)(b + L.off[L_MREF]);
    s.mprn = (uint8_t*)(b + L.off[L_MPRN]);
    s.manc = (uint8_t*)(b + L.off[L_MANC]);
    s.labels16 = (uint16_t*)(b + L.off[L_LAB16]);
    s.scratch16 = (uint16_t*)(b + L.off[L_SCR16]);
    s.mbits = (uint32_t*)(b + L.off[L_MBITS]);
    s.par = (int32_t*)(b + L.off[L_PAR]);
    s.cnt = (uint32_t*)(b + L.off[L_CNT]);
    s.rank = (int32_t*)(b + L.off[L_RANK]);
    s.szhist = (uint32_t*)(b + L.off[L_SZH]);
    s.roots = (int32_t*)(b + L.off[L_ROOTS]);
    s.list = (uint32_t*)(b + L.off[L_LIST]);
    s.tile_off = (uint32_t*)(b + L.off[L_TOFF]);
    s.lb = (unsigned long long*)(b + L.off[L_LB]);
    s.sparse = (int16_t*)(b + L.off[L_SPARSE]);
    s.rowf = (int16_t*)(b + L.off[L_ROWF]);
    s.dense = (int16_t*)(b + L.off[L_DENSE]);
    s.sc = (DevScalars*)(b + L.off[L_SC]);
    s.rbits = (uint32_t*)(b + L.off[L_RBITS]);
    s.sbits = (uint32_t*)(b + L.off[L_SBITS]);
    s.runroot = (int32_t*)(b + L.off[L_RUNR]);
    s.bord = (int32_t*)(b + L.off[L_BORD]);
    s.sbits_words = (int)(((size_t)W * H + 31) / 32);
    if (s.gexec) {
        cudaGraphExecDestroy(s.gexec);
        s.gexec = nullptr;
        s.gkey = GraphKey{};
    }
    return STK_OK;
}

Frame make_frame(const Slot& s, int W, int H, const stk_config* cfg) {
    Frame f{};
    f.W = W;
    f.H = H;
    f.P = s.P;
    f.N = (long long)W * H;
    f.TX = (W + kRowTile - 1) / kRowTile;
    f.n_tiles = H * f.TX;
    f.n_chunks = (f.n_tiles + kTilesPerChunk - 1) / kTilesPerChunk;
    f.bits_words = f.TX * 4;
    f.sms = s.sms;
    if (cfg) {
        f.kcfg = cfg->k;
        f.window = cfg->window;
        f.hw = cfg->window / 2;
        f.D = cfg->max_disparity;
        f.thr = cfg->threshold;
        f.frac = cfg->prune_fraction;
    }
    f.rgbL = s.rgbL;
    f.rgbR = s.rgbR;
    f.grayL = s.grayL;
    f.grayR = s.grayR;
    f.labels16 = s.labels16;
    f.mraw = s.mraw;
    f.mref = s.mref;
    f.mprn = nullptr;
    f.manc = nullptr;
    f.mbits = s.mbits;
    f.par = s.par;
    f.cnt = s.cnt;
    f.rank = s.rank;
    f.szhist = s.szhist;
    f.roots = s.roots;
    f.list = s.list;
    f.tile_off = s.tile_off;
    f.lb = s.lb;
    f.lb_stride = s.lb_stride;
    f.sparse = s.sparse;
    f.rowf = s.rowf;
    f.dense = s.dense;
    f.out_rgb = s.out_rgb;
    f.sc = s.sc;
    return f;
}

stk_status encode(stk_ctx* ctx, TMap& t, const void* ptr, int esz, int W, int H, int pitch_bytes,
                  int bw, int bh) {
    if (t.ptr == ptr && t.W == W && t.H == H && t.pitch == pitch_bytes && t.bw == bw &&
        t.bh == bh && t.esz == esz)
        return STK_OK;
    const cuuint64_t gdim[2] = {(cuuint64_t)W, (cuuint64_t)H};
    const cuuint64_t gstride[1] = {(cuuint64_t)pitch_bytes};
    const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = ctx->encode(&t.map, esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                    : CU_TENSOR_MAP_DATA_TYPE_UINT16,
                                   2, const_cast<void*>(ptr), gdim, gstride, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(ctx, STK_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    t.ptr = ptr;
    t.W = W;
    t.H = H;
    t.pitch = pitch_bytes;
    t.bw = bw;
    t.bh = bh;
    t.esz = esz;
    return STK_OK;
}

#define TRY(x)                          \
    do {                                \
        stk_status s_ = (x);            \
        if (s_ != STK_OK) return s_;    \
    } while (0)

// ----------------------------------------------------------- validation ---
stk_status check_config(stk_ctx* ctx, const stk_config* c) {
    if (!c) return fail(ctx, STK_EPARAM, "pipeline: null config");
    if (c->k < 1) return fail(ctx, STK_EPARAM, "pipeline: k must be at least 1, got " + std::to_string(c->k));
    if (c->window < 1 || c->window % 2 == 0)
        return fail(ctx, STK_EPARAM, "pipeline: window must be odd and positive, got " + std::to_string(c->window));
    if (c->max_disparity < 0)
        return fail(ctx, STK_EPARAM, "pipeline: max_disparity must be >= 0, got " + std::to_string(c->max_disparity));
    if (c->threshold < 0)
        return fail(ctx, STK_EPARAM, "pipeline: threshold must be >= 0, got " + std::to_string(c->threshold));
    if (!(c->prune_fraction >= 0.0 && c->prune_fraction < 1.0))
        return fail(ctx, STK_EPARAM, "pipeline: prune_fraction must be in [0, 1), got " + std::to_string(c->prune_fraction));
    if (c->workers < 1)
        return fail(ctx, STK_EPARAM, "pipeline: workers must be at least 1, got " + std::to_string(c->workers));
    return STK_OK;
}

stk_status check_focus(stk_ctx* ctx, const stk_focus* fo, int D, int* size_out) {
    if (fo->n_ranges <= 0 || !fo->lo || !fo->hi)
        return fail(ctx, STK_EPARAM, "build_blur_map: no focus ranges given");
    for (int i = 0; i < fo->n_ranges; ++i)
        if (fo->lo[i] < 0 || fo->lo[i] > fo->hi[i] || fo->hi[i] > D)
            return fail(ctx, STK_EPARAM, "build_blur_map: bad focus range [" + std::to_string(fo->lo[i]) +
                                             ", " + std::to_string(fo->hi[i]) + "] for max disparity " +
                                             std::to_string(D));
    const int size = fo->kernel_size > 0 ? fo->kernel_size : stk_default_kernel_size(fo->sigma);
    if (!(fo->sigma > 0.0))
        return fail(ctx, STK_EPARAM, "gaussian_kernel: sigma must be positive, got " + std::to_string(fo->sigma));
    if (size < 1 || size % 2 == 0)
        return fail(ctx, STK_EPARAM, "gaussian_kernel: size must be odd and positive, got " + std::to_string(size));
    *size_out = size;
    return STK_OK;
}

// Upload the focus LUT and blur weights for slot s (host-cached).
stk_status upload_focus(stk_ctx* ctx, Slot& s, const int* lo, const int* hi, int n, int D,
                        double sigma, int size, bool exact, BlurParams* bp) {
    const int lut_len = std::min(D, kMaxLut - 1) + 1;
    std::vector<uint8_t> lut(lut_len, 0);
    for (int d = 0; d < lut_len; ++d)
        for (int r = 0; r < n; ++r)
            if (d >= lo[r] && d <= hi[r]) lut[d] = 1;
    const int hw = size / 2;
    std::vector<float> g1(size);
    std::vector<double> g2((size_t)size * size);
    {
        double sum = 0.0;
        std::vector<double> t(size);
        for (int i = -hw; i <= hw; ++i) {
            t[i + hw] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma));
            sum += t[i + hw];
        }
        for (int i = 0; i < size; ++i) g1[i] = (float)(t[i] / sum);
        stk_gaussian_kernel(sigma, size, g2.data());
    }
    if (lut_len > s.lut_cap || (int)g2.size() > s.g_cap) {
        // the slot's stream may still read the old tables (a stage entry or a
        // frame); every captured graph holds their addresses -> drop it
        CK(cudaStreamSynchronize(s.st));
        if (s.gexec) {
            cudaGraphExecDestroy(s.gexec);
            s.gexec = nullptr;
            s.gkey = GraphKey{};
        }
    }
    if (lut_len > s.lut_cap) {
        if (s.d_lut) CK(cudaFree(s.d_lut));
        if (s.p_lut) CK(cudaFreeHost(s.p_lut));
        s.d_lut = nullptr;
        s.p_lut = nullptr;
        s.lut_cap = std::max(lut_len, 1024);
        CK(cudaMalloc(&s.d_lut, s.lut_cap));
        CK(cudaMallocHost(&s.p_lut, s.lut_cap));
        s.h_lut.clear();
    }
    if ((int)g2.size() > s.g_cap) {
        if (s.d_g1) CK(cudaFree(s.d_g1));
        if (s.d_g2) CK(cudaFree(s.d_g2));
        if (s.p_g1) CK(cudaFreeHost(s.p_g1));
        if (s.p_g2) CK(cudaFreeHost(s.p_g2));
        s.d_g1 = nullptr;
        s.d_g2 = nullptr;
        s.p_g1 = nullptr;
        s.p_g2 = nullptr;
        s.g_cap = std::max((int)g2.size(), 4096);
        CK(cudaMalloc(&s.d_g1, s.g_cap * sizeof(float)));
        CK(cudaMalloc(&s.d_g2, s.g_cap * sizeof(double)));
        CK(cudaMallocHost(&s.p_g1, s.g_cap * sizeof(float)));
        CK(cudaMallocHost(&s.p_g2, s.g_cap * sizeof(double)));
        s.h_g1.clear();
        s.h_g2.clear();
    }
    // A slot has at most one frame in flight and stage entries are
    // synchronous, so the previous copy out of the staging buffers has
    // completed by now; the new copies are ordered before this frame's kernels.
    if (s.h_lut != lut) {
        std::memcpy(s.p_lut, lut.data(), lut_len);
        CK(cudaMemcpyAsync(s.d_lut, s.p_lut, lut_len, cudaMemcpyHostToDevice, s.st));
        s.h_lut = lut;
    }
    if (s.h_g1 != g1 || s.h_g2 != g2) {
        std::memcpy(s.p_g1, g1.data(), g1.size() * sizeof(float));
        std::memcpy(s.p_g2, g2.data(), g2.size() * sizeof(double));
        CK(cudaMemcpyAsync(s.d_g1, s.p_g1, g1.size() * sizeof(float), cudaMemcpyHostToDevice, s.st));
        CK(cudaMemcpyAsync(s.d_g2, s.p_g2, g2.size() * sizeof(double), cudaMemcpyHostToDevice, s.st));
        s.h_g1 = g1;
        s.h_g2 = g2;
    }
    bp->hw = hw;
    bp->exact = exact ? 1 : 0;
    bp->g1 = s.d_g1;
    bp->g2 = s.d_g2;
    bp->sharp_lut = s.d_lut;
    bp->lut_len = lut_len;
    bp->blur_map = nullptr;
    return STK_OK;
}

// The global-memory blur fallback's float plane (12 bytes per pixel), only
// for separable kernels too wide for a shared-memory tile.
stk_status ensure_blur_scratch(stk_ctx* ctx, Slot& s, size_t N, BlurParams* bp) {
    bp->scratch = nullptr;
    if (!blur_needs_scratch(bp->hw, bp->exact != 0)) return STK_OK;
    const size_t need = 12 * std::max<size_t>(N, 1);
    if (need > s.blur_tmp_bytes) {
        CK(cudaStreamSynchronize(s.st));
        if (s.gexec) {  // a captured frame graph holds the old plane's address
            cudaGraphExecDestroy(s.gexec);
            s.gexec = nullptr;
            s.gkey = GraphKey{};
        }
        if (s.blur_tmp) CK(cudaFree(s.blur_tmp));
        s.blur_tmp = nullptr;
        CK(cudaMalloc(&s.blur_tmp, need));
        s.blur_tmp_bytes = need;
    }
    bp->scratch = s.blur_tmp;
    return STK_OK;
}

// --------------------------------------------------------- frame enqueue ---
// NVTX range for the host-side enqueue of one stage (SURVEY.md §5 tracing;
// free when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int enqueue_kernels(stk_ctx* ctx, Slot& s, const Frame& f, const BlurParams* bp, bool timed,
                    bool want_labels) {
    NvtxRange frame_range("stk enqueue frame");
    cudaStream_t st = s.st;
    int n = 0;
    static const char* kStage[8] = {"convert", "segment", "boundary", "match", "fill", "peek", "blur", "end"};
    auto rec = [&](int i) {
        if (timed) cudaEventRecord(s.ev[i], st);
        if (i > 0) nvtxRangePop();
        if (i < 7) nvtxRangePushA(kStage[i]);
    };
    cudaMemsetAsync(f.sc, 0, sizeof(DevScalars), st);
    cudaMemsetAsync(f.lb, 0, sizeof(unsigned long long) * LB_COUNT * f.lb_stride, st);
    rec(0);
    n += launch_lightness(f, ctx->d_tab, true, true, true, st, ctx->d_lut);  // left (+histogram), right
    rec(1);
    launch_kmeans(f, 0, 100, 0.5, st);
    ++n;
    if (want_labels) {
        launch_assign(f, f.grayL, f.labels16, st);
        ++n;
    }
    rec(2);
    // sparse starts all Unknown; the SAD kernels write the matchable pixels.
    // Lean frames skip the 2N-byte preset: the row fill reads the matchable
    // bits and takes every other pixel as unknown (full mode copies sparse out)
    const bool fill_masks = !f.full && fill_rows_masks(f.W);
    if (!fill_masks) cudaMemsetAsync(f.sparse, 0xff, (size_t)f.N * sizeof(int16_t), st);
    const bool want_list = sad_uses_list(f, ctx->sad_kernel);
    // B1, B2 (+ its overflow pass), B3 (+ B3b), B4-B7 (cooperative), B8 (+ list)
    n += launch_boundary_bits(f, s.rbits, s.runroot, s.bord, s.sbits, s.sbits_words, true, want_list, st);
    rec(3);
    if (f.W >= f.window && f.H >= f.window) {
        launch_sad(f, ctx->sad_kernel, &s.tm_sadL.map, &s.tm_sadR.map, st);
        ++n;
    }
    rec(4);
    launch_fill_rows(f, f.sparse, f.rowf, st, fill_masks ? f.mbits : nullptr);
    ++n;
    rec(5);
    launch_peek_cols(f, f.rowf, f.dense, nullptr, st);
    ++n;
    rec(6);
    if (bp) n += launch_blur(f, *bp, f.rgbL, f.out_rgb, f.dense, st);
    rec(7);
    cudaMemcpyAsync(s.h_sc, f.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st);
    return n;
}

bool want_full(const stk_frame_out* o) {
    return o && (o->left_lightness || o->right_lightness || o->labels || o->boundary_raw ||
                 o->boundary_refined || o->boundary_anchored || o->sparse || o->row_filled);
}

stk_status check_frame_args(stk_ctx* ctx, int slot, int w, int h, const stk_config* cfg,
                            const stk_focus* focus, int* ksize) {
    if (!ctx) return fail(ctx, STK_EPARAM, "stk: null context");
    if (slot < 0 || slot >= (int)ctx->slots.size())
        return fail(ctx, STK_EPARAM, "stk: slot " + std::to_string(slot) + " out of range");
    TRY(check_config(ctx, cfg));
    if (w < 0 || h < 0) return fail(ctx, STK_EPARAM, "pipeline: bad frame size " + dims(w, h));
    if ((long long)w * h == 0)  // k = min(cfg.k, 0 occupied bins) -> kmeans throws
        return fail(ctx, STK_EPARAM, "kmeans: k must be at least 1, got 0");
    const int margin = cfg->window / 2;
    if (2 * margin >= w)
        return fail(ctx, STK_EPARAM, "add_border_anchors: margin " + std::to_string(margin) +
                                         " does not fit in width " + std::to_string(w));
    if (w > 65535 || h > 65535)
        return fail(ctx, STK_EPARAM, "stk_b200: frame " + dims(w, h) + " exceeds 65535 per side");
    if (focus) TRY(check_focus(ctx, focus, cfg->max_disparity, ksize));
    if (ctx->slots[slot].pending)
        return fail(ctx, STK_EPARAM, "stk: slot " + std::to_string(slot) + " still has a frame in flight");
    return STK_OK;
}

// Common body of stk_frame_submit / stk_frame_submit_device.
stk_status submit(stk_ctx* ctx, int slot, const uint8_t* rgbL, const uint8_t* rgbR, bool host_in,
                  int w, int h, const stk_config* cfg, const stk_focus* focus,
                  const stk_frame_out* out, bool host_out, uint8_t* d_refocused, int16_t* d_dense,
                  bool timed) {
    NvtxRange range("stk_frame_submit");
    int ksize = 0;
    TRY(check_frame_args(ctx, slot, w, h, cfg, focus, &ksize));
    CK(cudaSetDevice(ctx->device));
    Slot& s = ctx->slots[slot];
    TRY(ensure_slot(ctx, s, w, h));
    Frame f = make_frame(s, w, h, cfg);
    const size_t N = (size_t)w * h;
    const bool full = host_out && want_full(out);
    f.full = full ? 1 : 0;
    if (full) {
        f.mprn = s.mprn;
        f.manc = s.manc;
    }
    if (!host_in) {
        f.rgbL = rgbL;
        f.rgbR = rgbR;
    }
    if (!host_out) {
        if (d_refocused) f.out_rgb = d_refocused;
        if (d_dense) f.dense = d_dense;
    }
    BlurParams bp{};
    if (focus) {
        TRY(upload_focus(ctx, s, focus->lo, focus->hi, focus->n_ranges, cfg->max_disparity,
                         focus->sigma, ksize, focus->exact_blur != 0, &bp));
        TRY(ensure_blur_scratch(ctx, s, N, &bp));
    }
    TRY(encode(ctx, s.tm_sadL, s.grayL, 1, w, h, s.P, 128, cfg->window));
    TRY(encode(ctx, s.tm_sadR, s.grayR, 1, w, h, s.P, 128, cfg->window));
    cudaStream_t st = s.st;
    if (host_in) {
        CK(cudaMemcpyAsync(s.rgbL, rgbL, 3 * N, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(s.rgbR, rgbR, 3 * N, cudaMemcpyHostToDevice, st));
    }
    const bool want_labels = full && out->labels;
    int nk = 0;
    bool graphed = false, captured = false;
    if (!timed && ctx->use_graphs) {
        GraphKey key;
        key.W = w;
        key.H = h;
        key.kcfg = cfg->k;
        key.window = cfg->window;
        key.D = cfg->max_disparity;
        key.thr = cfg->threshold;
        key.frac = cfg->prune_fraction;
        key.full = f.full;
        key.focus = focus ? 1 : 0;
        key.hw = bp.hw;
        key.exact = bp.exact;
        key.lut_len = bp.lut_len;
        key.sad = ctx->sad_kernel;
        key.want_raw = want_labels;
        key.rgbL = f.rgbL;
        key.rgbR = f.rgbR;
        key.out_rgb = f.out_rgb;
        key.dense = f.dense;
        key.lut = bp.sharp_lut;
        key.g1 = bp.g1;
        key.g2 = bp.g2;
        key.blur_tmp = bp.scratch;
        if (!(s.gexec && s.gkey == key)) {
            if (s.gexec) {
                cudaGraphExecDestroy(s.gexec);
                s.gexec = nullptr;
            }
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            s.kernels = enqueue_kernels(ctx, s, f, focus ? &bp : nullptr, false, want_labels);
            CK(cudaStreamEndCapture(st, &g));
            const cudaError_t ie = cudaGraphInstantiate(&s.gexec, g, 0);
            cudaGraphDestroy(g);
            CK(ie);
            s.gkey = key;
            captured = true;
        }
        CK(cudaGraphLaunch(s.gexec, st));
        nk = s.kernels;
        graphed = true;
    } else {
        nk = enqueue_kernels(ctx, s, f, focus ? &bp : nullptr, timed, want_labels);
        CK(cudaGetLastError());
    }
    if (host_out && out) {
        if (out->dense) CK(cudaMemcpyAsync(out->dense, f.dense, 2 * N, cudaMemcpyDeviceToHost, st));
        if (out->refocused && focus)
            CK(cudaMemcpyAsync(out->refocused, f.out_rgb, 3 * N, cudaMemcpyDeviceToHost, st));
        auto plane = [&](void* dst, const void* src) -> cudaError_t {
            return cudaMemcpy2DAsync(dst, w, src, s.P, w, h, cudaMemcpyDeviceToHost, st);
        };
        if (out->left_lightness) CK(plane(out->left_lightness, f.grayL));
        if (out->right_lightness) CK(plane(out->right_lightness, f.grayR));
        if (out->boundary_raw) CK(plane(out->boundary_raw, f.mraw));
        if (out->boundary_refined) CK(plane(out->boundary_refined, f.mprn));
        if (out->boundary_anchored) CK(plane(out->boundary_anchored, f.manc));
        if (out->labels) CK(cudaMemcpyAsync(out->labels, f.labels16, 2 * N, cudaMemcpyDeviceToHost, st));
        if (out->sparse) CK(cudaMemcpyAsync(out->sparse, f.sparse, 2 * N, cudaMemcpyDeviceToHost, st));
        if (out->row_filled) CK(cudaMemcpyAsync(out->row_filled, f.rowf, 2 * N, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(s.done, st));
    s.pending = true;
    s.timed = timed;
    s.graph = graphed;
    s.captured = captured;
    s.kernels = nk;
    s.f = f;
    s.out = (host_out && out) ? *out : stk_frame_out{};
    return STK_OK;
}

}  // namespace

// =================================================================== ABI ===
namespace stk {
void set_thread_error(const std::string& msg) { t_err = msg; }  // host I/O entries (stk_io.cpp)
}

extern "C" {

int stk_abi_version(void) { return STK_ABI_VERSION; }

int stk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

const char* stk_status_string(stk_status s) {
    switch (s) {
        case STK_OK: return "ok";
        case STK_EPARAM: return "parameter error";
        case STK_EIO: return "io error";
        case STK_EFORMAT: return "format error";
        case STK_ECUDA: return "cuda error";
        default: return "internal error";
    }
}

const char* stk_last_error(const stk_ctx* ctx) { return ctx ? ctx->err.c_str() : t_err.c_str(); }

stk_status stk_create(int device, int max_width, int max_height, int slots, stk_ctx** out) {
    stk_ctx* ctx = nullptr;
    if (!out) return fail(nullptr, STK_EPARAM, "stk_create: null out");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, STK_ECUDA, "stk_create: no CUDA device (this library has no CPU path)");
    if (device < 0 || device >= ndev)
        return fail(nullptr, STK_EPARAM, "stk_create: device " + std::to_string(device) + " out of range");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
        return fail(nullptr, STK_ECUDA, "stk_create: device is not sm_100 (Blackwell B200)");
    ctx = new stk_ctx();
    ctx->device = device;
    stk_status rc = STK_OK;
    do {
        if (cudaSetDevice(device) != cudaSuccess) {
            rc = fail(ctx, STK_ECUDA, "cudaSetDevice failed");
            break;
        }
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || !fn) {
            rc = fail(ctx, STK_ECUDA, "cuTensorMapEncodeTiled unavailable");
            break;
        }
        ctx->encode = (EncodeTiledFn)fn;
        std::unique_ptr<LstarTables> tabp(new LstarTables());
        LstarTables& tab = *tabp;
        make_lstar_tables(&tab);
        if (!lstar_buckets_ok(&tab)) {
            rc = fail(ctx, STK_EINTERNAL, "stk_create: L* bucket table has a bucket with 2 thresholds");
            break;
        }
        if (cudaMalloc(&ctx->d_tab, sizeof(LstarTables)) != cudaSuccess ||
            cudaMemcpy(ctx->d_tab, &tab, sizeof(tab), cudaMemcpyHostToDevice) != cudaSuccess) {
            rc = fail(ctx, STK_ECUDA, "stk_create: table upload failed");
            break;
        }
        // K1's exact 2^24-entry table, opt-in ($STK_LSTAR_LUT=1), persisting in
        // L2 for the slot streams below.  Measured at 4K: convert 52 -> 40 us on
        // the grey benchmark frames but 55 -> 93 us on uniformly random RGB
        // (L2 gathers), so the arithmetic kernel, flat across inputs, stays the
        // default.
        static const bool lut_on = [] {
            const char* e = getenv("STK_LSTAR_LUT");
            return e ? atoi(e) != 0 : false;
        }();
        if (lut_on) {
            if (cudaMalloc(&ctx->d_lut, size_t(1) << 24) != cudaSuccess) {
                rc = fail(ctx, STK_ECUDA, "stk_create: L* table allocation failed");
                break;
            }
            build_lstar_lut(ctx->d_tab, ctx->d_lut, 0);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                rc = fail(ctx, STK_ECUDA, "stk_create: L* table build failed");
                break;
            }
            int max_persist = 0;
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t want = std::min<size_t>(size_t(1) << 24, (size_t)max_persist);
            if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            cudaGetLastError();
        }
        cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
        ctx->slots.resize(std::max(slots, 1));
        for (Slot& s : ctx->slots) {
            s.sms = ctx->sms;
            if (cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreate(&s.done) != cudaSuccess ||
                cudaMallocHost(&s.h_sc, sizeof(DevScalars)) != cudaSuccess) {
                rc = fail(ctx, STK_ECUDA, "stk_create: stream/event setup failed");
                break;
            }
            for (auto& e : s.ev) cudaEventCreate(&e);
            const std::string nm = "stk dev" + std::to_string(device) + " slot " +
                                   std::to_string(&s - ctx->slots.data());
            nvtxNameCudaStreamA(s.st, nm.c_str());
            if (ctx->d_lut) {
                cudaStreamAttrValue av = {};
                av.accessPolicyWindow.base_ptr = ctx->d_lut;
                av.accessPolicyWindow.num_bytes = size_t(1) << 24;
                av.accessPolicyWindow.hitRatio = 1.0f;
                av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cudaStreamSetAttribute(s.st, cudaStreamAttributeAccessPolicyWindow, &av);
                cudaGetLastError();  // best effort: without persistence the table still works
            }
        }
        if (rc != STK_OK) break;
        if (max_width > 0 && max_height > 0) rc = ensure_slot(ctx, ctx->slots[0], max_width, max_height);
    } while (0);
    if (rc != STK_OK) {
        stk_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return STK_OK;
}

void stk_destroy(stk_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (Slot& s : ctx->slots) {
        if (s.st) cudaStreamSynchronize(s.st);
        if (s.gexec) cudaGraphExecDestroy(s.gexec);
        if (s.base) cudaFree(s.base);
        if (s.d_lut) cudaFree(s.d_lut);
        if (s.d_g1) cudaFree(s.d_g1);
        if (s.d_g2) cudaFree(s.d_g2);
        if (s.p_lut) cudaFreeHost(s.p_lut);
        if (s.p_g1) cudaFreeHost(s.p_g1);
        if (s.p_g2) cudaFreeHost(s.p_g2);
        if (s.blur_tmp) cudaFree(s.blur_tmp);
        if (s.cub_tmp) cudaFree(s.cub_tmp);
        if (s.h_sc) cudaFreeHost(s.h_sc);
        for (auto& e : s.ev)
            if (e) cudaEventDestroy(e);
        if (s.done) cudaEventDestroy(s.done);
        if (s.st) cudaStreamDestroy(s.st);
    }
    if (ctx->d_tab) cudaFree(ctx->d_tab);
    if (ctx->d_lut) cudaFree(ctx->d_lut);
    delete ctx;
}

stk_status stk_set_sad_kernel(stk_ctx* ctx, int kernel) {
    if (!ctx || kernel < 0 || kernel > 3) return fail(ctx, STK_EPARAM, "stk_set_sad_kernel: bad kernel");
    ctx->sad_kernel = kernel;
    for (Slot& s : ctx->slots) s.gkey = GraphKey{};
    return STK_OK;
}

stk_status stk_set_use_graphs(stk_ctx* ctx, int on) {
    if (!ctx) return fail(ctx, STK_EPARAM, "stk_set_use_graphs: null ctx");
    ctx->use_graphs = on ? 1 : 0;
    return STK_OK;
}

stk_status stk_host_alloc(size_t bytes, void** out) {
    stk_ctx* ctx = nullptr;
    CK(cudaMallocHost(out, bytes));
    return STK_OK;
}

void stk_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

stk_status stk_validate_config(const stk_config* cfg) { return check_config(nullptr, cfg); }

void stk_lstar_tables(double linear[256], double thr[256]) {
    std::unique_ptr<LstarTables> t(new LstarTables());
    make_lstar_tables(t.get());
    std::memcpy(linear, t->linear, sizeof(t->linear));
    std::memcpy(thr, t->thr, sizeof(t->thr));
}

int stk_default_kernel_size(double sigma) { return 2 * (int)std::ceil(3.0 * sigma) + 1; }

stk_status stk_gaussian_kernel(double sigma, int size, double* weights) {
    if (!(sigma > 0.0))
        return fail(nullptr, STK_EPARAM, "gaussian_kernel: sigma must be positive, got " + std::to_string(sigma));
    if (size < 1 || size % 2 == 0)
        return fail(nullptr, STK_EPARAM, "gaussian_kernel: size must be odd and positive, got " + std::to_string(size));
    const int h = size / 2;
    double sum = 0.0;
    for (int i = -h; i <= h; ++i)
        for (int j = -h; j <= h; ++j) {
            const double w = std::exp(-(i * i + j * j) / (2.0 * sigma * sigma));
            weights[(size_t)(i + h) * size + (j + h)] = w;
            sum += w;
        }
    for (size_t t = 0; t < (size_t)size * size; ++t) weights[t] /= sum;
    return STK_OK;
}

// ------------------------------------------------------------- frames -----
stk_status stk_frame_submit(stk_ctx* ctx, int slot, const uint8_t* rgb_left,
                            const uint8_t* rgb_right, int w, int h, const stk_config* cfg,
                            const stk_focus* focus, const stk_frame_out* out, int want_times) {
    return submit(ctx, slot, rgb_left, rgb_right, true, w, h, cfg, focus, out, true, nullptr,
                  nullptr, want_times != 0);
}

stk_status stk_frame_submit_device(stk_ctx* ctx, int slot, const uint8_t* d_rgb_left,
                                   const uint8_t* d_rgb_right, int w, int h,
                                   const stk_config* cfg, const stk_focus* focus,
                                   uint8_t* d_refocused, int16_t* d_dense, int want_times) {
    return submit(ctx, slot, d_rgb_left, d_rgb_right, false, w, h, cfg, focus, nullptr, false,
                  d_refocused, d_dense, want_times != 0);
}

stk_status stk_frame_wait(stk_ctx* ctx, int slot, stk_stats* stats, stk_times* times,
                          stk_frame_info* info) {
    if (!ctx || slot < 0 || slot >= (int)ctx->slots.size())
        return fail(ctx, STK_EPARAM, "stk_frame_wait: bad slot");
    Slot& s = ctx->slots[slot];
    if (!s.pending) return fail(ctx, STK_EPARAM, "stk_frame_wait: no frame in flight on slot");
    CK(cudaSetDevice(ctx->device));
    s.pending = false;
    CK(cudaEventSynchronize(s.done));
    CK(cudaGetLastError());
    const DevScalars& h = *s.h_sc;
    if (h.kerr) return fail(ctx, STK_EINTERNAL, "kmeans failed on device (code " + std::to_string(h.kerr) + ")");
    const double n = (double)s.f.N;
    if (stats) {
        stats->pixels = (uint64_t)s.f.N;
        stats->boundary_raw = h.raw_count;
        stats->boundary_refined = h.pruned_count;
        stats->matched = h.matched;
        stats->matched_fraction = n > 0 ? (double)h.matched / n : 0.0;
        stats->known_fraction = n > 0 ? (double)h.known / n : 0.0;
    }
    if (times) {
        std::memset(times, 0, sizeof(*times));
        if (s.timed) {
            float ms[7];
            for (int i = 0; i < 7; ++i) cudaEventElapsedTime(&ms[i], s.ev[i], s.ev[i + 1]);
            times->convert = ms[0];
            times->segment = ms[1];
            times->boundary = ms[2];
            times->match = ms[3];
            times->fill = ms[4];
            times->peek = ms[5];
            times->blur = ms[6];
        }
    }
    if (s.out.centers)
        for (int j = 0; j < 256; ++j) s.out.centers[j] = j < h.k ? h.centers[j] : 0.0;
    if (s.out.bin_assignment) std::memcpy(s.out.bin_assignment, h.assign16, 512);
    if (info) {
        info->sad_ops = h.sad_ops;
        info->components = h.n_roots;
        info->k = h.k;
        info->iterations_run = h.iters;
        info->kernels = s.kernels;
        info->graph = s.graph ? 1 : 0;
        info->captured = s.captured ? 1 : 0;
    }
    return STK_OK;
}

void* stk_slot_stream(stk_ctx* ctx, int slot) {
    if (!ctx || slot < 0 || slot >= (int)ctx->slots.size()) return nullptr;
    return (void*)ctx->slots[slot].st;
}

stk_status stk_run_frame(stk_ctx* ctx, const uint8_t* rgb_left, const uint8_t* rgb_right, int w,
                         int h, const stk_config* cfg, const stk_focus* focus,
                         const stk_frame_out* out, stk_stats* stats, stk_times* times) {
    TRY(stk_frame_submit(ctx, 0, rgb_left, rgb_right, w, h, cfg, focus, out, times != nullptr));
    return stk_frame_wait(ctx, 0, stats, times, nullptr);
}

// ---------------------------------------------------- per-stage entries ---
#define STAGE_BEGIN(w, h)                                                     \
    if (!ctx) return fail(ctx, STK_EPARAM, "stk: null context");              \
    if ((w) < 0 || (h) < 0) return fail(ctx, STK_EPARAM, "stk: bad size");    \
    CK(cudaSetDevice(ctx->device));                                           \
    Slot& s = ctx->slots[0];                                                  \
    if (s.pending) return fail(ctx, STK_EPARAM, "stk: slot 0 busy");          \
    TRY(ensure_slot(ctx, s, std::max((w), 1), std::max((h), 1)));             \
    Frame f = make_frame(s, (w), (h), nullptr);                               \
    const size_t N = (size_t)(w) * (h);                                       \
    cudaStream_t st = s.st;                                                   \
    (void)N;

#define H2D_PLANE(dst, src, esz)                                                              \
    if (N) CK(cudaMemcpy2DAsync((dst), (size_t)s.P * (esz), (src), (size_t)f.W * (esz),      \
                                (size_t)f.W * (esz), f.H, cudaMemcpyHostToDevice, st))
#define D2H_PLANE(dst, src, esz)                                                              \
    if (N) CK(cudaMemcpy2DAsync((dst), (size_t)f.W * (esz), (src), (size_t)s.P * (esz),      \
                                (size_t)f.W * (esz), f.H, cudaMemcpyDeviceToHost, st))
#define FINISH()                              \
    CK(cudaGetLastError());                   \
    CK(cudaStreamSynchronize(st));            \
    return STK_OK

stk_status stk_rgb_to_lightness(stk_ctx* ctx, const uint8_t* rgb, int w, int h, uint8_t* gray) {
    STAGE_BEGIN(w, h);
    if (N) CK(cudaMemcpyAsync(s.rgbL, rgb, 3 * N, cudaMemcpyHostToDevice, st));
    launch_lightness(f, ctx->d_tab, true, false, false, st);
    D2H_PLANE(gray, s.grayL, 1);
    FINISH();
}

stk_status stk_build_histogram(stk_ctx* ctx, const uint8_t* gray, int w, int h,
                               uint64_t counts[256]) {
    STAGE_BEGIN(w, h);
    H2D_PLANE(s.grayL, gray, 1);
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    launch_histogram(f, s.grayL, st);
    CK(cudaMemcpyAsync(s.h_sc, s.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    for (int v = 0; v < 256; ++v) counts[v] = s.h_sc->hist[v];
    return STK_OK;
}

stk_status stk_kmeans_histogram(stk_ctx* ctx, const uint64_t counts[256], int k, int max_iter,
                                double tol, double* centers, uint16_t bin_assignment[256],
                                int* iterations_run) {
    if (k < 1) return fail(ctx, STK_EPARAM, "kmeans: k must be at least 1, got " + std::to_string(k));
    if (max_iter < 1)
        return fail(ctx, STK_EPARAM, "kmeans: max_iter must be at least 1, got " + std::to_string(max_iter));
    int occ = 0;
    for (int v = 0; v < 256; ++v) occ += counts[v] > 0;
    if (occ == 0) return fail(ctx, STK_EPARAM, "kmeans: empty histogram");
    if (k > occ)
        return fail(ctx, STK_EPARAM, "kmeans: k=" + std::to_string(k) + " exceeds the " +
                                         std::to_string(occ) + " occupied bins");
    STAGE_BEGIN(1, 1);
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    CK(cudaMemcpyAsync(s.sc->hist, counts, 256 * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    launch_kmeans(f, k, max_iter, tol, st);
    CK(cudaMemcpyAsync(s.h_sc, s.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    if (s.h_sc->kerr) return fail(ctx, STK_EINTERNAL, "kmeans: device error");
    for (int j = 0; j < k; ++j) centers[j] = s.h_sc->centers[j];
    std::memcpy(bin_assignment, s.h_sc->assign16, 512);
    *iterations_run = s.h_sc->iters;
    return STK_OK;
}

stk_status stk_assign_pixels(stk_ctx* ctx, const uint8_t* gray, int w, int h,
                             const uint16_t bin_assignment[256], int k, uint16_t* labels) {
    if (k < 1) return fail(ctx, STK_EPARAM, "assign_pixels: clustering has no centers");
    STAGE_BEGIN(w, h);
    H2D_PLANE(s.grayL, gray, 1);
    CK(cudaMemcpyAsync(s.sc->assign16, bin_assignment, 512, cudaMemcpyHostToDevice, st));
    launch_assign(f, s.grayL, s.labels16, st);
    if (N) CK(cudaMemcpyAsync(labels, s.labels16, 2 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

// detect / fill / remove on the frame path's B1 kernel (k_morph_bits in stage
// mode: the same word-parallel morphology and edge rules the frame runs).
static stk_status morph_stage(stk_ctx* ctx, int mode, const void* in, int w, int h, uint8_t* out) {
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    const uint8_t* src;
    if (mode == MORPH_DETECT16) {
        H2D_PLANE(s.scratch16, in, 2);
        src = reinterpret_cast<const uint8_t*>(s.scratch16);
    } else {
        H2D_PLANE(s.mref, in, 1);
        src = s.mref;
    }
    launch_morph_stage_bits(f, mode, src, s.rbits, s.mraw, st);
    D2H_PLANE(out, s.mraw, 1);
    FINISH();
}

stk_status stk_detect_boundaries(stk_ctx* ctx, const uint16_t* labels, int w, int h,
                                 uint8_t* mask) {
    return morph_stage(ctx, MORPH_DETECT16, labels, w, h, mask);
}

stk_status stk_morph_fill(stk_ctx* ctx, const uint8_t* mask, int w, int h, uint8_t* out) {
    return morph_stage(ctx, MORPH_FILL, mask, w, h, out);
}

stk_status stk_morph_remove(stk_ctx* ctx, const uint8_t* mask, int w, int h, uint8_t* out) {
    return morph_stage(ctx, MORPH_REMOVE, mask, w, h, out);
}

stk_status stk_label_components(stk_ctx* ctx, const uint8_t* mask, int w, int h, int32_t* labels,
                                uint32_t* sizes, int32_t* by_size, size_t cap,
                                int* n_components) {
    STAGE_BEGIN(w, h);
    *n_components = 0;
    if (N == 0) return STK_OK;
    H2D_PLANE(s.mref, mask, 1);
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    f.frac = 0.0;
    // ComponentTable (boundary.hpp:39-45) from the frame path's run CCL
    // (k_bnd.cu B2/B3 + label kernels): canonical labels = rank of the
    // component's first pixel in raster order; sizes by label; by_size =
    // STABLE radix sort of the label ids by size, i.e. (size asc, label asc)
    // as boundary.cpp:136-146.  8-connected components are >= 2 px apart, so
    // C <= ceil(W/2) * ceil(H/2) ids fit the 2*P*H-byte scratch plane.
    uint32_t* d_sizes = s.szhist;                              // C
    int32_t* d_ids = reinterpret_cast<int32_t*>(s.scratch16);  // C
    int32_t* d_labels = reinterpret_cast<int32_t*>(s.list);    // N
    const size_t scan_need = label_components_tmp_bytes(s.sbits_words);
    if (scan_need > s.cub_bytes) {
        if (s.cub_tmp) CK(cudaFree(s.cub_tmp));
        s.cub_tmp = nullptr;
        CK(cudaMalloc(&s.cub_tmp, scan_need));
        s.cub_bytes = scan_need;
    }
    launch_label_components_bits(f, s.mref, s.rbits, s.runroot, s.bord, s.sbits, s.sbits_words,
                                 s.mbits, s.cub_tmp, s.cub_bytes, d_labels, d_sizes, d_ids, st);
    CK(cudaMemcpyAsync(s.h_sc, s.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    const int C = (int)s.h_sc->n_roots;
    if ((size_t)C > cap) return fail(ctx, STK_EPARAM, "label_components: capacity too small");
    CK(cudaMemcpyAsync(labels, d_labels, 4 * N, cudaMemcpyDeviceToHost, st));
    if (C > 0) {
        CK(cudaMemcpyAsync(sizes, d_sizes, 4 * (size_t)C, cudaMemcpyDeviceToHost, st));
        size_t need = 0;
        uint32_t* k_out = reinterpret_cast<uint32_t*>(s.roots);  // dense-id arrays: free now
        int32_t* v_out = reinterpret_cast<int32_t*>(s.cnt);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, need, d_sizes, k_out, d_ids, v_out, C, 0, 32, st));
        if (need > s.cub_bytes) {
            CK(cudaStreamSynchronize(st));
            if (s.cub_tmp) CK(cudaFree(s.cub_tmp));
            s.cub_tmp = nullptr;
            CK(cudaMalloc(&s.cub_tmp, need));
            s.cub_bytes = need;
        }
        CK(cub::DeviceRadixSort::SortPairs(s.cub_tmp, need, d_sizes, k_out, d_ids, v_out, C, 0, 32, st));
        CK(cudaMemcpyAsync(by_size, v_out, 4 * (size_t)C, cudaMemcpyDeviceToHost, st));
    }
    *n_components = C;
    FINISH();
}

stk_status stk_prune_components(stk_ctx* ctx, const uint8_t* mask, int w, int h, double fraction,
                                uint8_t* out) {
    if (!(fraction >= 0.0 && fraction < 1.0))
        return fail(ctx, STK_EPARAM, "prune_components: fraction must be in [0, 1), got " + std::to_string(fraction));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    H2D_PLANE(s.mref, mask, 1);
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    CK(cudaMemsetAsync(s.lb, 0, sizeof(unsigned long long) * LB_COUNT * s.lb_stride, st));
    f.frac = fraction;
    f.window = 1;
    f.hw = 0;
    f.mprn = s.mprn;
    f.manc = s.manc;
    // the frame path's bit-packed run CCL + prune (k_bnd.cu)
    launch_prune_mask_bits(f, s.mref, s.rbits, s.runroot, s.bord, s.sbits, s.sbits_words, st);
    D2H_PLANE(out, s.mprn, 1);
    FINISH();
}

stk_status stk_add_border_anchors(stk_ctx* ctx, const uint8_t* mask, int w, int h, int margin,
                                  uint8_t* out) {
    if (margin < 0 || 2 * margin >= w)
        return fail(ctx, STK_EPARAM, "add_border_anchors: margin " + std::to_string(margin) +
                                         " does not fit in width " + std::to_string(w));
    STAGE_BEGIN(w, h);
    H2D_PLANE(s.mref, mask, 1);
    launch_anchor_only(f, s.mref, s.manc, margin, st);
    D2H_PLANE(out, s.manc, 1);
    FINISH();
}

stk_status stk_sad_cost(stk_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                        int x, int y, int d, int window, uint32_t* cost) {
    const int hw = window / 2;
    if (window < 1 || window % 2 == 0)
        return fail(ctx, STK_EPARAM, "stereo: window must be odd and positive, got " + std::to_string(window));
    if (x - hw < 0 || x + hw >= w || y - hw < 0 || y + hw >= h || x - d - hw < 0 || x - d + hw >= w)
        return fail(ctx, STK_EPARAM, "sad_cost: window outside the images");
    STAGE_BEGIN(w, h);
    H2D_PLANE(s.grayL, left, 1);
    H2D_PLANE(s.grayR, right, 1);
    f.window = window;
    f.hw = hw;
    launch_sad_cost(f, x, y, d, s.tile_off, st);
    CK(cudaMemcpyAsync(cost, s.tile_off, 4, cudaMemcpyDeviceToHost, st));
    FINISH();
}

stk_status stk_match_boundary_pixels(stk_ctx* ctx, const uint8_t* left, const uint8_t* right,
                                     const uint8_t* mask, int w, int h, int window,
                                     int max_disparity, int16_t* out) {
    if (window < 1 || window % 2 == 0)
        return fail(ctx, STK_EPARAM, "stereo: window must be odd and positive, got " + std::to_string(window));
    if (max_disparity < 0)
        return fail(ctx, STK_EPARAM, "stereo: max_disparity must be >= 0, got " + std::to_string(max_disparity));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    H2D_PLANE(s.grayL, left, 1);
    H2D_PLANE(s.grayR, right, 1);
    H2D_PLANE(s.mref, mask, 1);
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    CK(cudaMemsetAsync(s.lb, 0, sizeof(unsigned long long) * LB_COUNT * s.lb_stride, st));
    f.window = window;
    f.hw = window / 2;
    f.D = max_disparity;
    TRY(encode(ctx, s.tm_sadL, s.grayL, 1, w, h, s.P, 128, window));
    TRY(encode(ctx, s.tm_sadR, s.grayR, 1, w, h, s.P, 128, window));
    launch_apply(f, false, st);
    if (w >= window && h >= window) launch_sad(f, ctx->sad_kernel, &s.tm_sadL.map, &s.tm_sadR.map, st);
    CK(cudaMemcpyAsync(out, s.sparse, 2 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

// dense_sad_baseline (evaluate.cpp:92-135): match_boundary_pixels with every
// pixel in the mask -- the mask plane is filled on the device.
stk_status stk_dense_sad_baseline(stk_ctx* ctx, const uint8_t* left, const uint8_t* right, int w,
                                  int h, int window, int max_disparity, int16_t* out) {
    if (window < 1 || window % 2 == 0)
        return fail(ctx, STK_EPARAM, "dense_sad_baseline: window must be odd and positive, got " +
                                         std::to_string(window));
    if (max_disparity < 0)
        return fail(ctx, STK_EPARAM, "dense_sad_baseline: max_disparity must be >= 0, got " +
                                         std::to_string(max_disparity));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    H2D_PLANE(s.grayL, left, 1);
    H2D_PLANE(s.grayR, right, 1);
    CK(cudaMemsetAsync(s.mref, 1, (size_t)s.P * h, st));
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    CK(cudaMemsetAsync(s.lb, 0, sizeof(unsigned long long) * LB_COUNT * s.lb_stride, st));
    f.window = window;
    f.hw = window / 2;
    f.D = max_disparity;
    TRY(encode(ctx, s.tm_sadL, s.grayL, 1, w, h, s.P, 128, window));
    TRY(encode(ctx, s.tm_sadR, s.grayR, 1, w, h, s.P, 128, window));
    launch_apply(f, false, st);
    if (w >= window && h >= window) launch_sad(f, ctx->sad_kernel, &s.tm_sadL.map, &s.tm_sadR.map, st);
    CK(cudaMemcpyAsync(out, s.sparse, 2 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

// bad_pixel_rate (evaluate.cpp:17-74)
stk_status stk_bad_pixel_rate(stk_ctx* ctx, const int16_t* computed, const int16_t* truth, int w,
                              int h, double delta_d, double* rate, uint64_t* compared,
                              uint64_t* excluded) {
    if (!(delta_d >= 0.0))
        return fail(ctx, STK_EPARAM, "bad_pixel_rate: delta_d must be >= 0, got " + std::to_string(delta_d));
    STAGE_BEGIN(w, h);
    unsigned long long counts[2] = {0, 0};
    if (N) {
        int16_t* d_c = s.sparse;
        int16_t* d_t = s.rowf;
        unsigned long long* d_out = &s.sc->raw_count;  // two adjacent u64 counters
        CK(cudaMemsetAsync(d_out, 0, 2 * sizeof(unsigned long long), st));
        CK(cudaMemcpyAsync(d_c, computed, 2 * N, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_t, truth, 2 * N, cudaMemcpyHostToDevice, st));
        launch_bad_pixel(d_c, d_t, (long long)N, delta_d, d_out, st);
        CK(cudaMemcpyAsync(counts, d_out, sizeof(counts), cudaMemcpyDeviceToHost, st));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
    if (compared) *compared = counts[0];
    if (excluded) *excluded = (uint64_t)N - counts[0];
    if (rate) *rate = counts[0] == 0 ? 0.0 : (double)counts[1] / (double)counts[0];
    return STK_OK;
}

// the match stage's brute-force ALU ceiling, microbenchmarked
stk_status stk_probe_sad_peak(stk_ctx* ctx, double* byte_ad_per_s) {
    if (!byte_ad_per_s) return fail(ctx, STK_EPARAM, "probe_sad_peak: null output");
    STAGE_BEGIN(1, 1);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const double rate = probe_vabsdiff4_rate(sms, reinterpret_cast<uint32_t*>(s.sc), st);
    CK(cudaGetLastError());
    if (rate <= 0.0) return fail(ctx, STK_ECUDA, "probe_sad_peak: probe kernel failed");
    *byte_ad_per_s = 4.0 * rate;
    return STK_OK;
}

stk_status stk_fill_scanlines(stk_ctx* ctx, const int16_t* sparse, int w, int h, int16_t* out) {
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    CK(cudaMemcpyAsync(s.sparse, sparse, 2 * N, cudaMemcpyHostToDevice, st));
    launch_fill_rows(f, s.sparse, s.rowf, st);
    CK(cudaMemcpyAsync(out, s.rowf, 2 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

stk_status stk_peek_columns(stk_ctx* ctx, const int16_t* map, int w, int h, int threshold,
                            int16_t* out) {
    if (threshold < 0)
        return fail(ctx, STK_EPARAM, "peek_columns: threshold must be >= 0, got " + std::to_string(threshold));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    CK(cudaMemcpyAsync(s.rowf, map, 2 * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(s.sc, 0, sizeof(DevScalars), st));
    f.thr = threshold;
    launch_peek_cols(f, s.rowf, s.dense, nullptr, st);
    CK(cudaMemcpyAsync(out, s.dense, 2 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

stk_status stk_build_blur_map(stk_ctx* ctx, const int16_t* depth, int w, int h, const int* lo,
                              const int* hi, int n_ranges, int max_disparity, uint8_t* map) {
    stk_focus fo{lo, hi, n_ranges, 1.0, 1, 0};
    int ks;
    TRY(check_focus(ctx, &fo, max_disparity, &ks));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    BlurParams bp{};
    TRY(upload_focus(ctx, s, lo, hi, n_ranges, max_disparity, 1.0, 1, false, &bp));
    CK(cudaMemcpyAsync(s.dense, depth, 2 * N, cudaMemcpyHostToDevice, st));
    launch_blur_map(f, s.dense, bp.sharp_lut, bp.lut_len, s.mraw, st);
    D2H_PLANE(map, s.mraw, 1);
    FINISH();
}

stk_status stk_selective_blur(stk_ctx* ctx, const uint8_t* rgb, const uint8_t* map, int w, int h,
                              double sigma, int size, int exact, uint8_t* out) {
    if (!(sigma > 0.0))
        return fail(ctx, STK_EPARAM, "gaussian_kernel: sigma must be positive, got " + std::to_string(sigma));
    if (size < 1 || size % 2 == 0)
        return fail(ctx, STK_EPARAM, "gaussian_kernel: size must be odd and positive, got " + std::to_string(size));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    const int lo0 = 0, hi0 = 0;
    BlurParams bp{};
    TRY(upload_focus(ctx, s, &lo0, &hi0, 1, 0, sigma, size, exact != 0, &bp));
    TRY(ensure_blur_scratch(ctx, s, N, &bp));
    bp.blur_map = s.mraw;
    CK(cudaMemcpyAsync(s.rgbL, rgb, 3 * N, cudaMemcpyHostToDevice, st));
    H2D_PLANE(s.mraw, map, 1);
    launch_blur(f, bp, s.rgbL, s.out_rgb, nullptr, st);
    CK(cudaMemcpyAsync(out, s.out_rgb, 3 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

stk_status stk_selective_blur_weights(stk_ctx* ctx, const uint8_t* rgb, const uint8_t* map, int w,
                                      int h, const double* weights, int size, uint8_t* out) {
    if (size < 1 || size % 2 == 0)
        return fail(ctx, STK_EPARAM, "selective_blur: kernel size must be odd and positive, got " +
                                         std::to_string(size));
    STAGE_BEGIN(w, h);
    if (N == 0) return STK_OK;
    const int lo0 = 0, hi0 = 0;
    BlurParams bp{};
    TRY(upload_focus(ctx, s, &lo0, &hi0, 1, 0, 1.0, size, true, &bp));
    // replace the Gaussian 2-D weights by the caller's (cache invalidated)
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(s.d_g2, weights, sizeof(double) * (size_t)size * size, cudaMemcpyHostToDevice));
    s.h_g2.clear();
    bp.blur_map = s.mraw;
    CK(cudaMemcpyAsync(s.rgbL, rgb, 3 * N, cudaMemcpyHostToDevice, st));
    H2D_PLANE(s.mraw, map, 1);
    launch_blur(f, bp, s.rgbL, s.out_rgb, nullptr, st);
    CK(cudaMemcpyAsync(out, s.out_rgb, 3 * N, cudaMemcpyDeviceToHost, st));
    FINISH();
}

}  // extern "C"
