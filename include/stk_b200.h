/*
 * stk_b200.h -- C-ABI of the B200-native (sm_100a) stereo depth + refocus
 * pipeline.  Plain pointers and sizes only; no C++ types, no exceptions cross
 * this boundary.  Every compute entry runs hand-written CUDA kernels; there is
 * no CPU fallback (a missing/unusable GPU returns STK_ECUDA).
 *
 * Each entry names the reference interface it replaces
 * (/root/reference/proj/include/stereotk/<header>:line).  The C++ shim
 * (include/stereotk/stereotk_b200.hpp, libstk_b200.so) re-implements the
 * stereotk:: value-type API on top of these entries, mapping STK_EPARAM to
 * stereotk::ParamError with the reference's message text.
 *
 * Layouts (all host buffers dense, row-major):
 *   RGB      w*h*3 bytes, interleaved        (image.hpp:11-33  RgbImage)
 *   gray     w*h bytes                       (image.hpp:35-53  GrayImage)
 *   labels   w*h uint16                      (segmentation.hpp:36-51 LabelMap)
 *   mask     w*h bytes, 0/1                  (boundary.hpp:11-33 BoundaryMask)
 *   disparity w*h int16, -1 = unknown        (stereo.hpp:13-40 DisparityMap)
 *
 * Threading: a context is not thread-safe; use one context per host thread
 * (and per GPU).  Contexts on different GPUs are independent.
 */
#ifndef STK_B200_H
#define STK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STK_ABI_VERSION 1

typedef enum stk_status {
    STK_OK = 0,
    STK_EPARAM = 1,    /* reference: stereotk::ParamError   (error.hpp:19-21) */
    STK_EIO = 2,       /* reference: stereotk::IoError      (error.hpp:9-11)  */
    STK_EFORMAT = 3,   /* reference: stereotk::FormatError  (error.hpp:14-16) */
    STK_ECUDA = 4,     /* CUDA runtime / device failure                        */
    STK_EINTERNAL = 5
} stk_status;

typedef struct stk_ctx stk_ctx;

/* stereotk::PipelineConfig (pipeline.hpp:18-25).  `workers` is validated
 * (>= 1) and otherwise ignored: the GPU result is identical for any value. */
typedef struct stk_config {
    int k;
    int window;
    int max_disparity;
    int threshold;
    double prune_fraction;
    int workers;
} stk_config;

/* stereotk::FocusSpec (refocus.hpp:23-26) + run_refocus_pipeline's
 * kernel_size (pipeline.hpp:85-89).  exact_blur = 1 selects the bit-exact
 * FP64 2-D blur; 0 (default) the separable FP32 blur (<= 1 LSB). */
typedef struct stk_focus {
    const int* lo;
    const int* hi;
    int n_ranges;
    double sigma;
    int kernel_size; /* <= 0: default_kernel_size(sigma) */
    int exact_blur;
} stk_focus;

/* stereotk::DepthStats (pipeline.hpp:42-49) */
typedef struct stk_stats {
    uint64_t pixels;
    uint64_t boundary_raw;
    uint64_t boundary_refined;
    uint64_t matched;
    double matched_fraction;
    double known_fraction;
} stk_stats;

/* stereotk::StageTimes (pipeline.hpp:28-39) in device milliseconds (CUDA
 * events), plus the blur stage the reference's bench omits. */
typedef struct stk_times {
    double convert, segment, boundary, match, fill, peek, blur;
} stk_times;

/* Extra per-frame facts (roofline inputs); not part of the reference API. */
typedef struct stk_frame_info {
    uint64_t sad_ops;      /* sum over matched pixels of (min(D, x-h)+1) * w^2 */
    uint64_t components;   /* connected components in the pre-prune mask */
    int k;                 /* effective clusters = min(cfg.k, occupied bins) */
    int iterations_run;
    int kernels;           /* kernel launches enqueued for this frame */
    int graph;             /* 1 if the frame ran as a CUDA graph */
    int captured;          /* 1 if this submit captured (re-instantiated) that graph */
} stk_frame_info;

/* Outputs of one frame (host pointers, or device pointers for the *_device
 * entries).  NULL = not wanted.  The lean outputs are `refocused` (needs a
 * focus) and `dense`; the rest are stereotk::DepthResult's intermediates
 * (pipeline.hpp:53-65) -- requesting any of them switches the frame to full
 * mode. */
typedef struct stk_frame_out {
    uint8_t* refocused;          /* 3N */
    int16_t* dense;              /* N  */
    uint8_t* left_lightness;     /* N  */
    uint8_t* right_lightness;    /* N  */
    double* centers;             /* 256 (first k valid) */
    uint16_t* bin_assignment;    /* 256 */
    uint16_t* labels;            /* N  */
    uint8_t* boundary_raw;       /* N  */
    uint8_t* boundary_refined;   /* N  (after fill, remove and prune) */
    uint8_t* boundary_anchored;  /* N  */
    int16_t* sparse;             /* N  */
    int16_t* row_filled;         /* N  */
} stk_frame_out;

/* ------------------------------------------------------------ lifecycle -- */
/* max_width/max_height size the first allocation (frames may be larger;
 * buffers then grow).  slots = frames in flight (>= 1). */
stk_status stk_create(int device, int max_width, int max_height, int slots, stk_ctx** out);
void stk_destroy(stk_ctx* ctx);
const char* stk_last_error(const stk_ctx* ctx); /* ctx may be NULL (thread-local) */
const char* stk_status_string(stk_status s);
int stk_abi_version(void);
/* CUDA devices visible to this process (0 without a GPU; never fails). */
int stk_device_count(void);
/* 0 = auto (3, else 2, else 1), 1 = per-pixel list kernel, 2 = column-sum strip
 * kernel, 3 = warp-specialised column-sum kernel (windows 9/15/21/31) */
stk_status stk_set_sad_kernel(stk_ctx* ctx, int kernel);
/* 1 = capture each frame's kernels in a CUDA graph and replay (default 1) */
stk_status stk_set_use_graphs(stk_ctx* ctx, int on);
stk_status stk_host_alloc(size_t bytes, void** out); /* pinned host memory */
void stk_host_free(void* p);

/* ----------------------------------------------- configuration checks -- */
/* validate_config (pipeline.hpp:91, pipeline.cpp:23-48) -- no GPU needed */
stk_status stk_validate_config(const stk_config* cfg);
/* default_kernel_size / gaussian_kernel (refocus.hpp:29-36) -- host side, as
 * in the reference (size^2 FP64 weights are a tiny host table). */
int stk_default_kernel_size(double sigma);
stk_status stk_gaussian_kernel(double sigma, int size, double* weights);
/* The host tables K1 uses (no GPU needed): linear[v] = srgb_to_linear(v)
 * (lightness.cpp:14-17) and thr[v] = smallest Y >= 0 whose 8-bit L* is >= v
 * (thr[0] = -1); gray(Y) = #{v >= 1 : thr[v] <= Y}. */
void stk_lstar_tables(double linear[256], double thr[256]);

/* ------------------------------------------ per-stage entries (parity) -- */
/* rgb_to_lightness (image.hpp:82) */
stk_status stk_rgb_to_lightness(stk_ctx* ctx, const uint8_t* rgb, int w, int h, uint8_t* gray);
/* build_histogram (segmentation.hpp:57) */
stk_status stk_build_histogram(stk_ctx* ctx, const uint8_t* gray, int w, int h,
                               uint64_t counts[256]);
/* kmeans_histogram (segmentation.hpp:67-68); centers capacity >= k */
stk_status stk_kmeans_histogram(stk_ctx* ctx, const uint64_t counts[256], int k, int max_iter,
                                double tol, double* centers, uint16_t bin_assignment[256],
                                int* iterations_run);
/* assign_pixels (segmentation.hpp:72); k = clustering.k() (0 -> EPARAM) */
stk_status stk_assign_pixels(stk_ctx* ctx, const uint8_t* gray, int w, int h,
                             const uint16_t bin_assignment[256], int k, uint16_t* labels);
/* detect_boundaries / morph_fill / morph_remove (boundary.hpp:51-62) */
stk_status stk_detect_boundaries(stk_ctx* ctx, const uint16_t* labels, int w, int h,
                                 uint8_t* mask);
stk_status stk_morph_fill(stk_ctx* ctx, const uint8_t* mask, int w, int h, uint8_t* out);
stk_status stk_morph_remove(stk_ctx* ctx, const uint8_t* mask, int w, int h, uint8_t* out);
/* label_components (boundary.hpp:65) -> ComponentTable (boundary.hpp:39-45).
 * labels: N int32; sizes/by_size: capacity `cap` (N is always enough);
 * *n_components receives C (EPARAM if cap < C). */
stk_status stk_label_components(stk_ctx* ctx, const uint8_t* mask, int w, int h, int32_t* labels,
                                uint32_t* sizes, int32_t* by_size, size_t cap,
                                int* n_components);
/* prune_components (boundary.hpp:71) */
stk_status stk_prune_components(stk_ctx* ctx, const uint8_t* mask, int w, int h, double fraction,
                                uint8_t* out);
/* add_border_anchors (boundary.hpp:77) */
stk_status stk_add_border_anchors(stk_ctx* ctx, const uint8_t* mask, int w, int h, int margin,
                                  uint8_t* out);
/* sad_cost (stereo.hpp:48-49); window must lie inside both views */
stk_status stk_sad_cost(stk_ctx* ctx, const uint8_t* left, const uint8_t* right, int w, int h,
                        int x, int y, int d, int window, uint32_t* cost);
/* match_boundary_pixels (stereo.hpp:58-62) */
stk_status stk_match_boundary_pixels(stk_ctx* ctx, const uint8_t* left, const uint8_t* right,
                                     const uint8_t* mask, int w, int h, int window,
                                     int max_disparity, int16_t* out);
/* fill_scanlines / peek_columns (reconstruct.hpp:13, 25-26) */
stk_status stk_fill_scanlines(stk_ctx* ctx, const int16_t* sparse, int w, int h, int16_t* out);
stk_status stk_peek_columns(stk_ctx* ctx, const int16_t* map, int w, int h, int threshold,
                            int16_t* out);
/* build_blur_map (refocus.hpp:42-43) */
stk_status stk_build_blur_map(stk_ctx* ctx, const int16_t* depth, int w, int h, const int* lo,
                              const int* hi, int n_ranges, int max_disparity, uint8_t* map);
/* selective_blur (refocus.hpp:50-51) with gaussian_kernel(sigma, size) */
stk_status stk_selective_blur(stk_ctx* ctx, const uint8_t* rgb, const uint8_t* map, int w, int h,
                              double sigma, int size, int exact, uint8_t* out);
/* selective_blur with arbitrary size x size weights (refocus.hpp:50-51,
 * GaussianKernel::weights): bit-exact FP64 2-D kernel, reference order. */
stk_status stk_selective_blur_weights(stk_ctx* ctx, const uint8_t* rgb, const uint8_t* map, int w,
                                      int h, const double* weights, int size, uint8_t* out);

/* ------------------------------------------------------ evaluation -- */
/* dense_sad_baseline (evaluate.hpp:35-36, evaluate.cpp:92-135): winner-takes-
 * all SAD over every pixel with a valid window (match_boundary_pixels with a
 * full mask). */
stk_status stk_dense_sad_baseline(stk_ctx* ctx, const uint8_t* left, const uint8_t* right, int w,
                                  int h, int window, int max_disparity, int16_t* out);
/* bad_pixel_rate (evaluate.hpp:22-24, evaluate.cpp:17-74): pixels known in
 * both maps are compared, bad iff |computed - truth| > delta_d; rate = bad /
 * compared (0 when nothing compared), excluded = w*h - compared. */
stk_status stk_bad_pixel_rate(stk_ctx* ctx, const int16_t* computed, const int16_t* truth, int w,
                              int h, double delta_d, double* rate, uint64_t* compared,
                              uint64_t* excluded);

/* Diagnostics: VABSDIFF4 throughput of this device in byte absolute
 * differences per second (4 per instruction), from a register-only probe
 * kernel -- the brute-force SAD ceiling the match stage is reported against
 * (SURVEY.md 8(d)); no reference counterpart. */
stk_status stk_probe_sad_peak(stk_ctx* ctx, double* byte_ad_per_s);

/* ----------------------------------------------------------- frames -- */
/* run_depth_pipeline (focus == NULL) / run_refocus_pipeline
 * (pipeline.hpp:78-89): synchronous, host buffers. */
stk_status stk_run_frame(stk_ctx* ctx, const uint8_t* rgb_left, const uint8_t* rgb_right, int w,
                         int h, const stk_config* cfg, const stk_focus* focus,
                         const stk_frame_out* out, stk_stats* stats, stk_times* times);
/* Asynchronous frame on `slot` (0 <= slot < slots): H2D of the pair, the
 * frame's kernels and D2H of the requested outputs are enqueued on the slot's
 * stream; host buffers must stay valid until stk_frame_wait.  Pinned host
 * memory (stk_host_alloc) makes the copies truly asynchronous. */
stk_status stk_frame_submit(stk_ctx* ctx, int slot, const uint8_t* rgb_left,
                            const uint8_t* rgb_right, int w, int h, const stk_config* cfg,
                            const stk_focus* focus, const stk_frame_out* out, int want_times);
/* Same with inputs and outputs already in device memory (no copies). */
stk_status stk_frame_submit_device(stk_ctx* ctx, int slot, const uint8_t* d_rgb_left,
                                   const uint8_t* d_rgb_right, int w, int h,
                                   const stk_config* cfg, const stk_focus* focus,
                                   uint8_t* d_refocused, int16_t* d_dense, int want_times);
stk_status stk_frame_wait(stk_ctx* ctx, int slot, stk_stats* stats, stk_times* times,
                          stk_frame_info* info);
/* The slot's cudaStream_t (as void*), for callers that time with events. */
void* stk_slot_stream(stk_ctx* ctx, int slot);

/* ------------------------------------------------------- file I/O -- */
/* Host-side file formats (no GPU needed).  Errors:
 * STK_EIO (cannot open / read / write, reference IoError) and STK_EFORMAT
 * (malformed or unsupported contents, reference FormatError), message via
 * stk_last_error(NULL).  Binary PGM/PPM exactly as image_io.cpp:29-241; PNG
 * decoded/encoded over zlib (the reference uses libpng, absent here).
 * Callers size buffers with stk_image_probe first; the load entries check
 * that w/h match the file (STK_EPARAM otherwise). */
/* width, height and channels (1 = P5 / grey PNG types, 3 = colour) */
stk_status stk_image_probe(const char* path, int* w, int* h, int* channels);
/* load_image (image.hpp:55-60, image_io.cpp:160-184): any supported file as
 * w*h*3 RGB; a P5 plane is replicated into the three channels. */
stk_status stk_load_image(const char* path, uint8_t* rgb, int w, int h);
/* load_gray (image.hpp:62-67, image_io.cpp:186-214): P5, or a PNG whose
 * pixels are grey.  The header comment lines (without "# ") are written to
 * `comments` joined by '\n' (may be NULL; *need = bytes required incl. NUL). */
stk_status stk_load_gray(const char* path, uint8_t* gray, int w, int h, char* comments, size_t cap,
                         size_t* need);
/* save_gray (image.hpp:69-72): P5; `comments` = '\n'-separated lines or NULL */
stk_status stk_save_gray(const char* path, const uint8_t* gray, int w, int h, const char* comments);
/* save_rgb (image.hpp:74-76): PNG when the extension is .png, else P6 */
stk_status stk_save_rgb(const char* path, const uint8_t* rgb, int w, int h);
/* save_disparity / load_disparity / load_ground_truth / disparity_mask_path
 * (evaluate.hpp:27-67, evaluate.cpp:76-90, 136-229) */
stk_status stk_save_disparity(const char* path, const int16_t* disparity, int w, int h,
                              double output_scale);
stk_status stk_load_disparity(const char* path, int16_t* disparity, int w, int h,
                              double fallback_scale);
stk_status stk_load_ground_truth(const char* path, int16_t* disparity, int w, int h, double scale);
stk_status stk_disparity_mask_path(const char* path, char* out, size_t cap, size_t* need);
/* Frame-pair discovery of the CLI (tools/main.cpp:247-284): every
 * <stem>_L.<ext> with a <stem>_R.<ext> beside it (ext .png/.ppm/.pgm), sorted
 * by stem, written as "left\tright\n" lines. */
stk_status stk_list_frame_pairs(const char* dir, char* out, size_t cap, size_t* need, int* count);

/* -------------------------------------------------- streamed frame I/O -- */
/* A directory of <stem>_L/_R pairs (stk_list_frame_pairs) refocused to
 * <out_dir>/<stem>.ppm|.png (and <stem>_disp.pgm when disparity_scale > 0):
 * decoder threads fill pinned host buffers ahead of the GPU, frames run on
 * `slots` GPU slots of `ctx` (stk_create with at least that many), writer
 * threads encode the results -- file decode, H2D, kernels, D2H and encode all
 * overlap.  Frames shard across processes by index:
 * this call handles frames f with f % shard_count == shard_index.  No
 * reference counterpart (its CLI runs one pair per process,
 * tools/main.cpp:327-379); each output equals run_refocus_pipeline's. */
typedef struct stk_video_opts {
    int slots;            /* GPU frames in flight (<= the context's slots) */
    int decode_threads;   /* host decoder threads */
    int write_threads;    /* host encoder threads */
    int png;              /* 1: write .png, 0: .ppm */
    double disparity_scale; /* > 0: also save_disparity(dense, <stem>_disp.pgm, scale) */
    int shard_index, shard_count;
} stk_video_opts;
typedef struct stk_video_report {
    int frames;           /* frames this call processed */
    int frames_total;     /* pairs in the directory */
    double wall_s, frames_per_s;
    double decode_s, write_s, gpu_wait_s; /* summed thread time per phase */
    double matched_fraction;
} stk_video_report;
stk_status stk_video_refocus(stk_ctx* ctx, const char* in_dir, const char* out_dir, const stk_config* cfg,
                             const stk_focus* focus, const stk_video_opts* opts, stk_video_report* report);

#ifdef __cplusplus
}
#endif
#endif /* STK_B200_H */
