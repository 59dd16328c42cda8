// stk_internal.cuh -- types shared by the sm_100a kernels and the C-ABI host
// code.  One stereo frame lives in HBM as the planes below (see DESIGN.md
// "Data layout in HBM").  8-bit planes are row-pitched (pitch P, a multiple of
// 64 bytes, as TMA needs 16-byte strides); 16/32-bit planes are dense with
// index y*W+x, so a union-find root index IS the raster index the reference's
// discovery order is defined on (boundary.cpp:96-107).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

namespace stk {

constexpr int kRowTile = 128;         // columns per row-tile (compaction + SAD list tiles)
constexpr int kTilesPerWarp = 4;      // consecutive row-tiles one warp compacts
constexpr int kTilesPerChunk = 32;    // row-tiles per look-back chunk (8 warps x 4)
constexpr uint32_t kRemoved = 0x80000000u;  // prune flag OR-ed into cnt[root]

// Counters for the single-pass decoupled look-back scans.
enum LookbackUse { LB_ROOTS = 0, LB_RANK = 1, LB_LIST = 2, LB_SAD = 3, LB_COUNT = 4 };

// Frame-wide scalars, device resident; zeroed (cudaMemsetAsync) at frame start.
struct DevScalars {
    unsigned long long hist[256];      // left-lightness histogram (K1)
    double centers[256];               // K-Means centers (K2)
    unsigned short assign16[256];      // bin_assignment (K2)
    unsigned char lut[256];            // gray -> cluster index (K2, k <= 256)
    int k;                             // min(cfg.k, occupied)   (pipeline.cpp:76-80)
    int iters;                         // iterations_run
    int kerr;                          // 1: empty histogram, 2: k > occupied, 3: k < 1
    int pad0;
    unsigned long long raw_count;      // boundary_raw.count()
    unsigned long long refined_count;  // after fill + remove (prune input)
    unsigned long long pruned_count;   // boundary_refined.count() (after prune)
    unsigned long long matched;        // M = list length (sparse.known_count())
    unsigned long long known;          // dense.known_count()
    unsigned long long sad_ops;        // sum over list of (d_lim+1)*w*w (roofline)
    unsigned long long budget;         // floor(fraction * refined_count)
    unsigned long long s_star;         // prune: sizes < s_star go ...
    unsigned long long q;              // ... and the first q of size s_star
    unsigned int n_roots;              // component count C
    unsigned int n_list;               // == matched
    unsigned int n_lroots;             // tile-local roots (K4a -> K4c)
    unsigned int n_ovf;                // B2 regions with a tile of > 256 runs (second pass)
    unsigned int ctr[LB_COUNT];        // dynamic chunk counters
    unsigned int psel_done;            // prune select: finished blocks
    unsigned int gbar_count;           // grid barrier (cooperative prune kernel)
    unsigned int gbar_gen;
    unsigned int n_edges;              // B3 -> B3b border edge list length
    unsigned int united;               // 1: B3b did the prune's compress + root stats (B4, B5)
    unsigned int pruned;               // 1: B3b also did the prune's select + classes (B6, B7)
    unsigned long long psel[128];      // prune select: per-block pixel sums
    unsigned long long gsum[512];      // cooperative prune: per-block pixel sums
    unsigned int gcnt[512];            // cooperative prune: per-block size-s* root counts
};

// Everything a kernel needs to know about one frame, passed by value.
struct Frame {
    int W, H, P;        // width, height, pitch of u8 planes (bytes)
    long long N;        // W*H
    int TX;             // row-tiles per row = ceil(W / kRowTile)
    int n_tiles;        // H * TX
    int n_chunks;       // ceil(n_tiles / kTilesPerChunk)
    int bits_words;     // u32 words per row of the matchable bit-mask
    int sms;            // SM count of the context's device (grid sizing)
    // configuration (PipelineConfig, pipeline.hpp:18-25)
    int kcfg, window, hw, D, thr;
    double frac;
    int full;           // write every DepthResult intermediate
    // planes
    const uint8_t* rgbL;
    const uint8_t* rgbR;
    uint8_t* grayL;
    uint8_t* grayR;
    uint16_t* labels16;   // full mode only (dense)
    uint8_t* mraw;        // raw boundary (pitched)
    uint8_t* mref;        // after fill+remove (pitched)
    uint8_t* mprn;        // after prune (pitched, full mode only)
    uint8_t* manc;        // anchored (pitched, full mode only)
    uint32_t* mbits;      // matchable bits (anchored & window fits), bits_words per row
    int32_t* par;         // union-find parent / root index (dense)
    uint32_t* cnt;        // component size at root index (dense)
    int32_t* rank;        // canonical component label at root index (dense)
    uint32_t* szhist;     // component-size histogram (N + 2)
    int32_t* roots;       // root raster indices in raster order (C)
    uint32_t* list;       // matchable pixels (y << 16 | x) in raster order (M)
    uint32_t* tile_off;   // list offset of each row-tile (n_tiles + 1)
    unsigned long long* lb;  // look-back status words, LB_COUNT * lb_stride
    int lb_stride;
    int16_t* sparse;
    int16_t* rowf;
    int16_t* dense;
    uint8_t* out_rgb;
    DevScalars* sc;
};

// Host-side constant tables for K1 (computed with the host libm, see
// stk_capi.cu: linear[] = srgb_to_linear, thr[v] = smallest Y with L*(Y) >= v).
struct LstarTables {
    double linear[256];
    double thr[256];   // thr[0] = -1 (always passes), thr[1..255] ascending
    // Bucketed form used by K1: for Y in [b/4096, (b+1)/4096),
    // gray = base[b] + (Y >= tb[b]); every bucket holds at most one threshold
    // (checked on the host; the minimum threshold spacing is 4.3e-4 > 1/4096).
    double tb[4097];
    unsigned char base[4097];
    // prod[c][v] = coefficient_c * linear[v] (lightness.cpp:41-43 products,
    // IEEE round-to-nearest on the host == __dmul_rn on the device)
    double prod[3][256];
    // packed bucket words for K1's shared-memory lookup: base[b] << 24 | q[b],
    // q[b] = floor(2^24 * (4096 * tb[b] - b)) (0xffffff without a threshold);
    // a Y in bucket b with floor(2^24 * (4096 * Y - b)) != q[b] decides
    // Y >= tb[b] from the integers alone (all steps exact), ties read tb[b].
    alignas(16) uint32_t bw[4097];
    // fprod[c][v] = (float)prod[c][v] (round to nearest): K1's FP32 screen
    float fprod[3][256];
    // K1's screen table: sub[s] = the gray of every Y within 2^-20 of the
    // sub-bucket [s 2^-16, (s+1) 2^-16) when no threshold lies in that span,
    // else 0xff; bright = bits of 1 + (thr[255] + 2^-20) rounded up: a
    // screened Y' at or above it is gray 255 (0xff in sub[] too)
    alignas(16) uint8_t sub[65536];
    uint32_t bright;
};
constexpr int kLstarBuckets = 4096;

// ---------------------------------------------------------------- launchers --
// Every launcher enqueues on `st` and never synchronises.  Implementations in
// k_*.cu.
// returns the number of kernels launched
int launch_lightness(const Frame& f, const LstarTables* dtab, bool left, bool right,
                     bool hist, cudaStream_t st, const uint8_t* lut = nullptr);
// the exact 2^24-entry L* table (lut[r << 16 | g << 8 | b]) used by the frame path
void build_lstar_lut(const LstarTables* dtab, uint8_t* lut, cudaStream_t st);
void launch_histogram(const Frame& f, const uint8_t* gray, cudaStream_t st);
void launch_kmeans(const Frame& f, int k_fixed, int max_iter, double tol, cudaStream_t st);
void launch_assign(const Frame& f, const uint8_t* gray, uint16_t* out, cudaStream_t st);

// stage modes of the frame path's B1 kernel (k_bnd.cu MB_*)
enum MorphMode { MORPH_DETECT16 = 1, MORPH_FILL = 2, MORPH_REMOVE = 3 };

// Bit-packed boundary stage of the frame path (k_bnd.cu): morphology from
// gray, run-based CCL, prune, anchors, matchable bits and frame counts
// (+ raw / pruned / anchored bytes in full mode; + the SAD list if asked).
// Returns the number of kernels launched.
int launch_boundary_bits(const Frame& f, uint32_t* rbits, int32_t* runroot, int32_t* bord,
                          uint32_t* sbits, int sbits_words, bool anchors, bool want_list,
                          cudaStream_t st);
// B2-B8 alone on refined bits already in rbits (refined_count set); returns the kernel count
int launch_ccl_prune_bits(const Frame& f, uint32_t* rbits, int32_t* runroot, int32_t* bord,
                           uint32_t* sbits, int sbits_words, bool anchors, cudaStream_t st);
// stage entries detect_boundaries / morph_fill / morph_remove on B1
void launch_morph_stage_bits(const Frame& f, int mode, const uint8_t* src, uint32_t* rbits,
                             uint8_t* out, cudaStream_t st);  // B1 in stage mode (k_bnd.cu)
void launch_label_components_bits(const Frame& f, const uint8_t* mask, uint32_t* rbits, int32_t* runroot,
                                  int32_t* bord, uint32_t* gbits, int gbits_words, uint32_t* wscan,
                                  void* tmp, size_t tmp_bytes, int32_t* labels, uint32_t* sizes,
                                  int32_t* ids, cudaStream_t st);  // run CCL labels (k_bnd.cu)
size_t label_components_tmp_bytes(int gbits_words);
// bytes of the region border-label buffer (B2 / B3, k_bnd.cu) for a W x H frame
size_t bord_bytes(int W, int H);
// stage entry prune_components on a pitched byte mask (writes f.mprn / f.manc)
void launch_prune_mask_bits(const Frame& f, const uint8_t* mask, uint32_t* rbits, int32_t* runroot,
                            int32_t* bord, uint32_t* sbits, int sbits_words, cudaStream_t st);
// K9 evaluation: out[0] += compared, out[1] += bad (evaluate.cpp:17-74)
// VABSDIFF4 instructions per second on this device (probe kernel, blocking)
double probe_vabsdiff4_rate(int sms, uint32_t* scratch, cudaStream_t st);
void launch_bad_pixel(const int16_t* comp, const int16_t* truth, long long n, double delta,
                      unsigned long long* out, cudaStream_t st);
// true when launch_sad will run the per-pixel list kernel (it needs f.list)
bool sad_uses_list(const Frame& f, int kernel);
// stage entries: byte mask (f.mref) -> matchable bits + list (k_apply.cu)
void launch_apply(const Frame& f, bool anchors, cudaStream_t st);
void launch_anchor_only(const Frame& f, const uint8_t* in, uint8_t* out, int margin, cudaStream_t st);
size_t sad_list_smem_bytes(int window, int D);
size_t blur_smem_bytes(int hw, bool exact);
void launch_sad_cost(const Frame& f, int x, int y, int d, uint32_t* out, cudaStream_t st);

enum SadKernel { SAD_AUTO = 0, SAD_LIST = 1, SAD_STRIP = 2, SAD_WS = 3 };
// K5b column-sum strip kernel; returns false (nothing launched) when the
// configuration is outside its register/shared-memory envelope.
bool launch_sad_strip(const Frame& f, cudaStream_t st, bool dry = false);
// K5c warp-specialised column-sum kernel (windows 9/15/21/31); false when
// outside its envelope.
bool launch_sad_ws(const Frame& f, cudaStream_t st, bool dry = false);
void launch_sad(const Frame& f, int kernel, const CUtensorMap* tmL, const CUtensorMap* tmR,
                cudaStream_t st);
// mbits (frame path, k_fill_rows16p only): pixels outside it read as unknown,
// so sparse needs no -1 preset; fill_rows_masks(W) says whether it applies
void launch_fill_rows(const Frame& f, const int16_t* in, int16_t* out, cudaStream_t st,
                      const uint32_t* mbits = nullptr);
bool fill_rows_masks(int W);
void launch_peek_cols(const Frame& f, const int16_t* in, int16_t* out, int16_t* seg_scratch,
                      cudaStream_t st);
size_t peek_scratch_bytes(int W, int H);

struct BlurParams {
    int hw;              // kernel half width (size / 2)
    int exact;           // 1: FP64 2-D in the reference's summation order
    const float* g1;     // separable 1-D weights (size), device
    const double* g2;    // 2-D weights (size*size), device (exact mode)
    const uint8_t* sharp_lut;  // sharp_lut[d] for d in [0, lut_len)
    int lut_len;
    const uint8_t* blur_map;   // if non-null: explicit map (stage entry), pitched P
    float* scratch;            // 3 floats per pixel: vertical sums of the global-memory
                               // fallback for kernels too wide for a shared-memory tile
};
// true when launch_blur needs bp.scratch (separable kernel beyond the tiles)
bool blur_needs_scratch(int hw, bool exact);
int launch_blur(const Frame& f, const BlurParams& bp, const uint8_t* in_rgb, uint8_t* out_rgb,
                const int16_t* depth, cudaStream_t st);  // returns the launches
void launch_blur_map(const Frame& f, const int16_t* depth, const uint8_t* sharp_lut,
                     int lut_len, uint8_t* out, cudaStream_t st);

}  // namespace stk
