/*
 * stk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the stereotk per-frame pipeline
 * (reference: /root/reference/proj/src/<stage>.cpp).  It exists so that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg have a checker that
 * travels to the GPU box (where /root/reference does not exist).  It is never
 * linked into, loaded by or called from the product library
 * (paper_2001_07809_b200/); the product path fails loudly without its CUDA
 * extension.
 *
 * Parity of this restatement is pinned in tests/test_oracle_cpu.py against
 *   (1) the reference compiled from its own sources (oracle/_ref, see
 *       oracle/Makefile) whenever that library is present, and
 *   (2) the committed golden fixtures in tests/golden/ generated from the
 *       compiled reference by tests/golden/make_golden.py.
 *
 * All images are dense row-major arrays: RGB = w*h*3 interleaved bytes,
 * gray/mask = w*h bytes, labels = w*h u16, disparity = w*h i16 (-1 unknown).
 * Functions return 0 on success and a negative code on a parameter error
 * (the reference throws stereotk::ParamError in those cases).
 */
#ifndef STK_ORACLE_H
#define STK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_EPARAM (-1)

/* lightness.cpp:25-53 */
void orc_lightness(const uint8_t* rgb, int w, int h, uint8_t* gray);
/* segmentation.cpp:11-44 */
void orc_histogram(const uint8_t* gray, size_t n, uint64_t counts[256]);
/* segmentation.cpp:64-144; returns ORC_EPARAM on the reference's throws */
int orc_kmeans(const uint64_t counts[256], int k, int max_iter, double tol,
               double* centers, uint16_t bin_assignment[256],
               int* iterations_run);
/* segmentation.cpp:146-155 */
void orc_assign(const uint8_t* gray, size_t n, const uint16_t bin_assignment[256],
                uint16_t* labels);
/* boundary.cpp:11-85 */
void orc_detect(const uint16_t* labels, int w, int h, uint8_t* out);
void orc_fill(const uint8_t* mask, int w, int h, uint8_t* out);
void orc_remove(const uint8_t* mask, int w, int h, uint8_t* out);
/* boundary.cpp:87-148.  labels: w*h i32; sizes/by_size: capacity w*h.
 * Returns the component count. */
int orc_label_components(const uint8_t* mask, int w, int h, int32_t* labels,
                         uint32_t* sizes, int32_t* by_size);
/* boundary.cpp:150-178 */
int orc_prune(const uint8_t* mask, int w, int h, double fraction, uint8_t* out);
/* boundary.cpp:180-195 */
int orc_anchors(const uint8_t* mask, int w, int h, int margin, uint8_t* out);
/* stereo.cpp:12-28 */
uint32_t orc_sad_cost(const uint8_t* left, const uint8_t* right, int w, int x,
                      int y, int d, int window);
/* stereo.cpp:62-102 */
int orc_match(const uint8_t* left, const uint8_t* right, const uint8_t* mask,
              int w, int h, int window, int max_disparity, int16_t* out);
/* reconstruct.cpp:11-33 */
void orc_fill_scanlines(const int16_t* sparse, int w, int h, int16_t* out);
/* reconstruct.cpp:40-109 */
int orc_peek_columns(const int16_t* map, int w, int h, int threshold,
                     int16_t* out);
/* refocus.cpp:12-43 */
int orc_default_kernel_size(double sigma);
int orc_gaussian_kernel(double sigma, int size, double* weights);
/* refocus.cpp:45-73 */
int orc_blur_map(const int16_t* depth, int w, int h, const int* lo,
                 const int* hi, int n_ranges, int max_disparity, uint8_t* map);
/* refocus.cpp:75-113 */
void orc_selective_blur(const uint8_t* rgb, const uint8_t* map, int w, int h,
                        const double* weights, int size, uint8_t* out);

/* pipeline.cpp:50-134 + 136-151 */
typedef struct {
    int k, window, max_disparity, threshold;
    double prune_fraction;
} orc_config;

typedef struct {
    uint64_t pixels, boundary_raw, boundary_refined, matched;
    double matched_fraction, known_fraction;
} orc_stats;

/* Every intermediate of one frame (DepthResult, pipeline.hpp:53-65).  Any
 * pointer may be NULL except `dense`. */
typedef struct {
    uint8_t *left_lightness, *right_lightness;
    double* centers; /* 256 */
    uint16_t* bin_assignment; /* 256 */
    int k, iterations_run;
    uint16_t* labels;
    uint8_t *boundary_raw, *boundary_refined, *boundary_anchored;
    int16_t *sparse, *row_filled, *dense;
} orc_depth;

int orc_run_depth(const uint8_t* rgb_left, const uint8_t* rgb_right, int w,
                  int h, const orc_config* cfg, orc_depth* out,
                  orc_stats* stats, double stage_ms[6]);
int orc_run_refocus(const uint8_t* rgb_left, const uint8_t* rgb_right, int w,
                    int h, const orc_config* cfg, const int* lo, const int* hi,
                    int n_ranges, double sigma, int kernel_size,
                    uint8_t* refocused, orc_depth* depth, orc_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
