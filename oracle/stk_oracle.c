/*
 * stk_oracle.c -- TEST INFRASTRUCTURE ONLY (see stk_oracle.h).
 *
 * Single-threaded C restatement of the reference stage semantics.  Each
 * function cites the reference lines it follows; the arithmetic order of
 * every floating-point expression is kept exactly (build with
 * -ffp-contract=off, no -march=native) so results are bit-identical to the
 * reference built the same way on the same libm.
 */
#define _POSIX_C_SOURCE 199309L
#include "stk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* ---------------------------------------------------------------- L* ---- */

/* lightness.cpp:14-17 (inverse sRGB companding) */
static double srgb_to_linear(int v) {
    const double c = v / 255.0;
    return c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
}

/* lightness.cpp:25-53: Y evaluated left to right without contraction, then
 * L* = 116 f - 16, scaled by 255/100, lround, clamp to [0,255]. */
void orc_lightness(const uint8_t* rgb, int w, int h, uint8_t* gray) {
    const double eps = 216.0 / 24389.0, kappa = 24389.0 / 27.0;
    double lin[256];
    for (int v = 0; v < 256; ++v) lin[v] = srgb_to_linear(v);
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        const uint8_t* p = rgb + 3 * i;
        const double y = 0.2126 * lin[p[0]] + 0.7152 * lin[p[1]] + 0.0722 * lin[p[2]];
        const double f = y > eps ? cbrt(y) : (kappa * y + 16.0) / 116.0;
        const double lstar = 116.0 * f - 16.0;
        long s = lround(lstar * 255.0 / 100.0);
        if (s < 0) s = 0;
        if (s > 255) s = 255;
        gray[i] = (uint8_t)s;
    }
}

/* ------------------------------------------------------- segmentation ---- */

/* segmentation.cpp:11-44 (partial histograms sum to the same counts) */
void orc_histogram(const uint8_t* gray, size_t n, uint64_t counts[256]) {
    memset(counts, 0, 256 * sizeof(uint64_t));
    for (size_t i = 0; i < n; ++i) counts[gray[i]]++;
}

/* segmentation.cpp:49-60: nearest center, ties to the lowest index */
static int nearest(const double* c, int k, double v) {
    int best = 0;
    double bd = fabs(v - c[0]);
    for (int j = 1; j < k; ++j) {
        const double d = fabs(v - c[j]);
        if (d < bd) { bd = d; best = j; }
    }
    return best;
}

/* segmentation.cpp:64-144 */
int orc_kmeans(const uint64_t counts[256], int k, int max_iter, double tol,
               double* centers, uint16_t bin_assignment[256], int* iterations_run) {
    if (k < 1 || max_iter < 1) return ORC_EPARAM;           /* :66-73 */
    int lo = -1, hi = -1, occupied = 0;
    for (int v = 0; v < 256; ++v)
        if (counts[v]) { if (lo < 0) lo = v; hi = v; ++occupied; }
    if (occupied == 0 || k > occupied) return ORC_EPARAM;   /* :85-93 */
    if (k == 1) centers[0] = (lo + hi) / 2.0;               /* :96-102 */
    else
        for (int j = 0; j < k; ++j) centers[j] = lo + (hi - lo) * (j / (k - 1.0));
    int asg[256];
    uint64_t wsum[256], vsum[256];
    *iterations_run = 0;
    for (int it = 1; it <= max_iter; ++it) {                /* :104-136 */
        for (int v = 0; v < 256; ++v) asg[v] = nearest(centers, k, v);
        memset(wsum, 0, sizeof(wsum));
        memset(vsum, 0, sizeof(vsum));
        for (int v = 0; v < 256; ++v) {
            if (!counts[v]) continue;
            wsum[asg[v]] += counts[v];
            vsum[asg[v]] += counts[v] * (uint64_t)v;
        }
        double move = 0.0;
        for (int j = 0; j < k; ++j) {
            if (!wsum[j]) continue;                          /* empty keeps */
            const double upd = (double)vsum[j] / (double)wsum[j];
            const double m = fabs(upd - centers[j]);
            if (move < m) move = m;                          /* std::max */
            centers[j] = upd;
        }
        *iterations_run = it;
        if (move < tol) break;
    }
    for (int v = 0; v < 256; ++v)                            /* :139-142 */
        bin_assignment[v] = (uint16_t)nearest(centers, k, v);
    return 0;
}

/* segmentation.cpp:146-155 */
void orc_assign(const uint8_t* gray, size_t n, const uint16_t bin_assignment[256],
                uint16_t* labels) {
    for (size_t i = 0; i < n; ++i) labels[i] = bin_assignment[gray[i]];
}

/* ----------------------------------------------------------- boundary ---- */

/* boundary.cpp:11-39: 1 iff an in-image Moore neighbour has another label */
void orc_detect(const uint16_t* lab, int w, int h, uint8_t* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const uint16_t c = lab[(size_t)y * w + x];
            int b = 0;
            for (int dy = -1; dy <= 1 && !b; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int nx = x + dx, ny = y + dy;
                    if ((dx || dy) && nx >= 0 && nx < w && ny >= 0 && ny < h &&
                        lab[(size_t)ny * w + nx] != c) { b = 1; break; }
                }
            out[(size_t)y * w + x] = (uint8_t)b;
        }
}

#define M(a, x, y) ((a)[(size_t)(y) * w + (x)])

/* boundary.cpp:41-63: interior 0 with all eight neighbours set becomes 1 */
void orc_fill(const uint8_t* m, int w, int h, uint8_t* out) {
    memcpy(out, m, (size_t)w * h);
    if (w < 3 || h < 3) return;
    for (int y = 1; y < h - 1; ++y)
        for (int x = 1; x < w - 1; ++x)
            if (!M(m, x, y) && M(m, x - 1, y - 1) && M(m, x, y - 1) && M(m, x + 1, y - 1) &&
                M(m, x - 1, y) && M(m, x + 1, y) && M(m, x - 1, y + 1) && M(m, x, y + 1) &&
                M(m, x + 1, y + 1))
                M(out, x, y) = 1;
}

/* boundary.cpp:65-85: interior 1 with all four 4-neighbours set becomes 0 */
void orc_remove(const uint8_t* m, int w, int h, uint8_t* out) {
    memcpy(out, m, (size_t)w * h);
    if (w < 3 || h < 3) return;
    for (int y = 1; y < h - 1; ++y)
        for (int x = 1; x < w - 1; ++x)
            if (M(m, x, y) && M(m, x, y - 1) && M(m, x - 1, y) && M(m, x + 1, y) &&
                M(m, x, y + 1))
                M(out, x, y) = 0;
}

static int32_t uf_find(int32_t* p, int32_t i) {
    while (p[i] != i) { p[i] = p[p[i]]; i = p[i]; }
    return i;
}

static const uint32_t* g_sort_sizes;
static int cmp_by_size(const void* a, const void* b) {
    const int32_t la = *(const int32_t*)a, lb = *(const int32_t*)b;
    if (g_sort_sizes[la] != g_sort_sizes[lb]) return g_sort_sizes[la] < g_sort_sizes[lb] ? -1 : 1;
    return la < lb ? -1 : (la > lb);
}

/* boundary.cpp:87-148.  Restated with union-find: the reference's raster
 * discovery order of a component equals the raster order of its smallest
 * pixel index, so labels are the ranks of min-index roots.  by_size sorts by
 * (size, label), boundary.cpp:136-146. */
int orc_label_components(const uint8_t* m, int w, int h, int32_t* labels,
                         uint32_t* sizes, int32_t* by_size) {
    const size_t n = (size_t)w * h;
    int32_t* p = (int32_t*)malloc(n * sizeof(int32_t) + 1);
    for (size_t i = 0; i < n; ++i) p[i] = (int32_t)i;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            if (!M(m, x, y)) continue;
            const int32_t i = y * w + x;
            const int nx[4] = {x - 1, x - 1, x, x + 1}, ny[4] = {y, y - 1, y - 1, y - 1};
            for (int t = 0; t < 4; ++t) {
                if (nx[t] < 0 || nx[t] >= w || ny[t] < 0 || !M(m, nx[t], ny[t])) continue;
                int32_t a = uf_find(p, i), b = uf_find(p, ny[t] * w + nx[t]);
                if (a != b) { if (a < b) p[b] = a; else p[a] = b; }
            }
        }
    int nc = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!m[i]) { labels[i] = -1; continue; }
        const int32_t r = uf_find(p, (int32_t)i);
        if (r == (int32_t)i) { labels[i] = nc; sizes[nc] = 0; ++nc; }
        else labels[i] = labels[r];          /* r < i: already labelled */
        sizes[labels[i]]++;
    }
    free(p);
    for (int c = 0; c < nc; ++c) by_size[c] = c;
    g_sort_sizes = sizes;
    qsort(by_size, (size_t)nc, sizeof(int32_t), cmp_by_size);
    return nc;
}

/* boundary.cpp:150-178: remove smallest-first while removed+size <= budget */
int orc_prune(const uint8_t* m, int w, int h, double fraction, uint8_t* out) {
    if (!(fraction >= 0.0 && fraction < 1.0)) return ORC_EPARAM;
    const size_t n = (size_t)w * h;
    int32_t* lab = (int32_t*)malloc(n * sizeof(int32_t) + 1);
    uint32_t* sz = (uint32_t*)malloc(n * sizeof(uint32_t) + 4);
    int32_t* bys = (int32_t*)malloc(n * sizeof(int32_t) + 4);
    uint8_t* rm = (uint8_t*)calloc(n + 1, 1);
    const int nc = orc_label_components(m, w, h, lab, sz, bys);
    uint64_t count = 0;
    for (size_t i = 0; i < n; ++i) count += m[i];
    const double budget = fraction * (double)count;
    uint64_t removed = 0;
    for (int t = 0; t < nc; ++t) {
        const int32_t c = bys[t];
        if ((double)(removed + sz[c]) > budget) break;
        removed += sz[c];
        rm[c] = 1;
    }
    for (size_t i = 0; i < n; ++i) out[i] = (lab[i] >= 0 && rm[lab[i]]) ? 0 : m[i];
    free(lab); free(sz); free(bys); free(rm);
    return 0;
}

/* boundary.cpp:180-195 */
int orc_anchors(const uint8_t* m, int w, int h, int margin, uint8_t* out) {
    if (margin < 0 || 2 * margin >= w) return ORC_EPARAM;
    memcpy(out, m, (size_t)w * h);
    for (int y = margin; y <= h - 1 - margin; ++y) {
        M(out, margin, y) = 1;
        M(out, w - 1 - margin, y) = 1;
    }
    return 0;
}

/* ------------------------------------------------------------- stereo ---- */

/* stereo.cpp:12-28 */
uint32_t orc_sad_cost(const uint8_t* L, const uint8_t* R, int w, int x, int y,
                      int d, int window) {
    const int hw = window / 2;
    uint32_t s = 0;
    for (int dy = -hw; dy <= hw; ++dy) {
        const uint8_t* l = L + (size_t)(y + dy) * w + (x - hw);
        const uint8_t* r = R + (size_t)(y + dy) * w + (x - d - hw);
        for (int i = 0; i < window; ++i) s += (uint32_t)abs((int)l[i] - (int)r[i]);
    }
    return s;
}

/* stereo.cpp:62-102 (validation :32-58 is size/parameter checks) */
int orc_match(const uint8_t* L, const uint8_t* R, const uint8_t* mask, int w,
              int h, int window, int max_disparity, int16_t* out) {
    if (window < 1 || window % 2 == 0 || max_disparity < 0) return ORC_EPARAM;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) out[i] = -1;
    const int hw = window / 2;
    if (w < window || h < window) return 0;
    for (int y = hw; y < h - hw; ++y)
        for (int x = hw; x < w - hw; ++x) {
            if (!M(mask, x, y)) continue;
            const int dl = max_disparity < x - hw ? max_disparity : x - hw;
            uint32_t best = 0xFFFFFFFFu;
            int bd = 0;
            for (int d = 0; d <= dl; ++d) {
                const uint32_t c = orc_sad_cost(L, R, w, x, y, d, window);
                if (c < best) { best = c; bd = d; }   /* strict: ties keep small d */
            }
            M(out, x, y) = (int16_t)bd;
        }
    return 0;
}

/* -------------------------------------------------------- reconstruct ---- */

/* reconstruct.cpp:11-33: fill between consecutive equal knowns (snapshot) */
void orc_fill_scanlines(const int16_t* s, int w, int h, int16_t* out) {
    memcpy(out, s, (size_t)w * h * sizeof(int16_t));
    for (int y = 0; y < h; ++y) {
        int px = -1;
        int16_t pd = -1;
        for (int x = 0; x < w; ++x) {
            const int16_t d = M(s, x, y);
            if (d < 0) continue;
            if (px >= 0 && d == pd)
                for (int f = px + 1; f < x; ++f) M(out, f, y) = d;
            px = x;
            pd = d;
        }
    }
}

/* reconstruct.cpp:40-46 */
static int16_t peek_estimate(int16_t a, int16_t b, int thr) {
    const int r = a >= b ? a - b : b - a;
    if (r > thr) return a < b ? a : b;
    return (int16_t)((a + b) / 2);
}

/* reconstruct.cpp:50-109 */
int orc_peek_columns(const int16_t* map, int w, int h, int thr, int16_t* out) {
    if (thr < 0) return ORC_EPARAM;
    memcpy(out, map, (size_t)w * h * sizeof(int16_t));
    int* rows = (int*)malloc(sizeof(int) * (size_t)(h + 1));
    int16_t* ds = (int16_t*)malloc(sizeof(int16_t) * (size_t)(h + 1));
    for (int x = 0; x < w; ++x) {
        int n = 0;
        for (int y = 0; y < h; ++y)
            if (M(map, x, y) >= 0) { rows[n] = y; ds[n] = M(map, x, y); ++n; }
        if (n == 0) continue;
        if (n == 1) {
            for (int y = 0; y < h; ++y) if (M(map, x, y) < 0) M(out, x, y) = ds[0];
            continue;
        }
        int next = 0;
        for (int y = 0; y < h; ++y) {
            while (next < n && rows[next] <= y) ++next;
            if (M(map, x, y) >= 0) continue;
            const int lo = next == 0 ? 0 : (next == n ? n - 2 : next - 1);
            M(out, x, y) = peek_estimate(ds[lo], ds[lo + 1], thr);
        }
    }
    free(rows);
    free(ds);
    return 0;
}

/* ------------------------------------------------------------ refocus ---- */

/* refocus.cpp:12-14 */
int orc_default_kernel_size(double sigma) { return 2 * (int)ceil(3.0 * sigma) + 1; }

/* refocus.cpp:16-43 */
int orc_gaussian_kernel(double sigma, int size, double* wts) {
    if (!(sigma > 0.0) || size < 1 || size % 2 == 0) return ORC_EPARAM;
    const int hh = size / 2;
    double sum = 0.0;
    for (int i = -hh; i <= hh; ++i)
        for (int j = -hh; j <= hh; ++j) {
            const double v = exp(-(i * i + j * j) / (2.0 * sigma * sigma));
            wts[(size_t)(i + hh) * size + (j + hh)] = v;
            sum += v;
        }
    for (size_t t = 0; t < (size_t)size * size; ++t) wts[t] /= sum;
    return 0;
}

/* refocus.cpp:45-73 */
int orc_blur_map(const int16_t* depth, int w, int h, const int* lo, const int* hi,
                 int nr, int max_disparity, uint8_t* map) {
    if (nr <= 0) return ORC_EPARAM;
    for (int r = 0; r < nr; ++r)
        if (lo[r] < 0 || lo[r] > hi[r] || hi[r] > max_disparity) return ORC_EPARAM;
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        const int16_t d = depth[i];
        int sharp = 0;
        if (d >= 0)
            for (int r = 0; r < nr && !sharp; ++r) sharp = d >= lo[r] && d <= hi[r];
        map[i] = sharp ? 0 : 1;
    }
    return 0;
}

static inline int clampi(int v, int a, int b) { return v < a ? a : (v > b ? b : v); }

/* refocus.cpp:75-113: 2-D FP64 accumulation, i outer / j inner, replicate */
void orc_selective_blur(const uint8_t* img, const uint8_t* map, int w, int h,
                        const double* wts, int size, uint8_t* out) {
    memcpy(out, img, (size_t)w * h * 3);
    const int hh = size / 2;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            if (!map[(size_t)y * w + x]) continue;
            double acc[3] = {0.0, 0.0, 0.0};
            for (int i = -hh; i <= hh; ++i) {
                const int sy = clampi(y + i, 0, h - 1);
                for (int j = -hh; j <= hh; ++j) {
                    const int sx = clampi(x + j, 0, w - 1);
                    const double wt = wts[(size_t)(i + hh) * size + (j + hh)];
                    const uint8_t* p = img + ((size_t)sy * w + sx) * 3;
                    acc[0] += wt * p[0];
                    acc[1] += wt * p[1];
                    acc[2] += wt * p[2];
                }
            }
            for (int c = 0; c < 3; ++c) {
                long v = lround(acc[c]);
                out[((size_t)y * w + x) * 3 + c] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
            }
        }
}

/* ----------------------------------------------------------- pipeline ---- */

static int validate(const orc_config* c) {                  /* pipeline.cpp:23-48 */
    if (c->k < 1 || c->window < 1 || c->window % 2 == 0 || c->max_disparity < 0 ||
        c->threshold < 0 || !(c->prune_fraction >= 0.0 && c->prune_fraction < 1.0))
        return ORC_EPARAM;
    return 0;
}

static void* take(void* p, size_t bytes, void** own) {
    if (p) return p;
    *own = malloc(bytes + 16);
    return *own;
}

/* pipeline.cpp:50-134 */
int orc_run_depth(const uint8_t* rl, const uint8_t* rr, int w, int h,
                  const orc_config* cfg, orc_depth* o, orc_stats* st,
                  double stage_ms[6]) {
    if (validate(cfg)) return ORC_EPARAM;
    const size_t n = (size_t)w * h;
    void* own[11] = {0};
    uint8_t* gl = (uint8_t*)take(o->left_lightness, n, &own[0]);
    uint8_t* gr = (uint8_t*)take(o->right_lightness, n, &own[1]);
    uint16_t* lab = (uint16_t*)take(o->labels, 2 * n, &own[2]);
    uint8_t* braw = (uint8_t*)take(o->boundary_raw, n, &own[3]);
    uint8_t* bref = (uint8_t*)take(o->boundary_refined, n, &own[4]);
    uint8_t* banc = (uint8_t*)take(o->boundary_anchored, n, &own[5]);
    int16_t* sp = (int16_t*)take(o->sparse, 2 * n, &own[6]);
    int16_t* rf = (int16_t*)take(o->row_filled, 2 * n, &own[7]);
    uint8_t* tmp = (uint8_t*)malloc(n + 16);
    double cbuf[256];
    uint16_t abuf[256];
    double* centers = o->centers ? o->centers : cbuf;
    uint16_t* asg = o->bin_assignment ? o->bin_assignment : abuf;
    double t0 = now_ms(), t1;
    int rc = 0;

    orc_lightness(rl, w, h, gl);
    orc_lightness(rr, w, h, gr);
    t1 = now_ms(); if (stage_ms) stage_ms[0] = t1 - t0; t0 = t1;

    uint64_t hist[256];
    orc_histogram(gl, n, hist);
    int occ = 0;
    for (int v = 0; v < 256; ++v) occ += hist[v] > 0;
    const int k = cfg->k < occ ? cfg->k : occ;                /* :76-80 */
    rc = orc_kmeans(hist, k, 100, 0.5, centers, asg, &o->iterations_run);
    if (rc) goto done;
    o->k = k;
    orc_assign(gl, n, asg, lab);
    t1 = now_ms(); if (stage_ms) stage_ms[1] = t1 - t0; t0 = t1;

    orc_detect(lab, w, h, braw);
    orc_fill(braw, w, h, tmp);
    orc_remove(tmp, w, h, bref);
    memcpy(tmp, bref, n);
    orc_prune(tmp, w, h, cfg->prune_fraction, bref);
    rc = orc_anchors(bref, w, h, cfg->window / 2, banc);
    if (rc) goto done;
    t1 = now_ms(); if (stage_ms) stage_ms[2] = t1 - t0; t0 = t1;

    rc = orc_match(gl, gr, banc, w, h, cfg->window, cfg->max_disparity, sp);
    if (rc) goto done;
    t1 = now_ms(); if (stage_ms) stage_ms[3] = t1 - t0; t0 = t1;
    orc_fill_scanlines(sp, w, h, rf);
    t1 = now_ms(); if (stage_ms) stage_ms[4] = t1 - t0; t0 = t1;
    rc = orc_peek_columns(rf, w, h, cfg->threshold, o->dense);
    t1 = now_ms(); if (stage_ms) stage_ms[5] = t1 - t0;

    if (st) {                                                 /* :121-132 */
        memset(st, 0, sizeof(*st));
        st->pixels = n;
        for (size_t i = 0; i < n; ++i) {
            st->boundary_raw += braw[i];
            st->boundary_refined += bref[i];
            st->matched += sp[i] >= 0;
        }
        if (n) {
            uint64_t known = 0;
            for (size_t i = 0; i < n; ++i) known += o->dense[i] >= 0;
            st->matched_fraction = (double)st->matched / (double)n;
            st->known_fraction = (double)known / (double)n;
        }
    }
done:
    free(tmp);
    for (int i = 0; i < 11; ++i) free(own[i]);
    return rc;
}

/* pipeline.cpp:136-151 */
int orc_run_refocus(const uint8_t* rl, const uint8_t* rr, int w, int h,
                    const orc_config* cfg, const int* lo, const int* hi, int nr,
                    double sigma, int kernel_size, uint8_t* out, orc_depth* depth,
                    orc_stats* st) {
    const size_t n = (size_t)w * h;
    orc_depth local;
    memset(&local, 0, sizeof(local));
    orc_depth* d = depth ? depth : &local;
    int16_t* own_dense = NULL;
    if (!d->dense) d->dense = own_dense = (int16_t*)malloc(2 * n + 16);
    int rc = orc_run_depth(rl, rr, w, h, cfg, d, st, NULL);
    uint8_t* map = (uint8_t*)malloc(n + 16);
    double* wts = NULL;
    if (!rc) rc = orc_blur_map(d->dense, w, h, lo, hi, nr, cfg->max_disparity, map);
    if (!rc) {
        const int size = kernel_size > 0 ? kernel_size : orc_default_kernel_size(sigma);
        wts = (double*)malloc(sizeof(double) * (size_t)size * size + 8);
        rc = orc_gaussian_kernel(sigma, size, wts);
        if (!rc) orc_selective_blur(rl, map, w, h, wts, size, out);
    }
    free(map);
    free(wts);
    if (own_dense) { free(own_dense); d->dense = NULL; }
    return rc;
}
