/*
 * synth.c -- deterministic synthetic stereo inputs (host side, plain C).
 *
 * Not part of the per-frame hot path: these generators produce the benchmark
 * and test inputs.  All randomness is raw std::mt19937 draws (restated here as
 * a 32-bit Mersenne Twister seeded exactly like std::mt19937(seed)), so every
 * scene is byte-identical to what the reference's own generators produce
 * (reference: proj/tests/synthetic.cpp:11-127; pinned against the compiled
 * reference in tests/test_oracle_cpu.py).
 *
 *   G1 = stk_synth_bench_frame            (synthetic.cpp:106-127)
 *   G2 = stk_synth_dead_leaves            (the
 *        paper-density "dead leaves" scene: ~18 % boundary pixels)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t s[624];
    int i;
} mt_t;

static void mt_seed(mt_t* m, uint32_t seed) {
    m->s[0] = seed;
    for (int k = 1; k < 624; ++k)
        m->s[k] = 1812433253u * (m->s[k - 1] ^ (m->s[k - 1] >> 30)) + (uint32_t)k;
    m->i = 624;
}

static uint32_t mt_next(mt_t* m) {
    if (m->i >= 624) {
        for (int k = 0; k < 624; ++k) {
            const uint32_t y = (m->s[k] & 0x80000000u) | (m->s[(k + 1) % 624] & 0x7fffffffu);
            m->s[k] = m->s[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        m->i = 0;
    }
    uint32_t y = m->s[m->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

uint32_t stk_synth_mt_draw(uint32_t seed, int skip) {
    mt_t m;
    mt_seed(&m, seed);
    for (int i = 0; i < skip; ++i) mt_next(&m);
    return mt_next(&m);
}

void stk_synth_raw_words(uint32_t seed, size_t n, uint32_t* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt_next(&m);
}

void stk_synth_random_rgb(int w, int h, uint32_t seed, uint8_t* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (size_t i = 0; i < (size_t)w * h * 3; ++i) out[i] = (uint8_t)(mt_next(&m) & 0xFFu);
}

void stk_synth_random_gray(int w, int h, uint32_t seed, uint8_t* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (size_t i = 0; i < (size_t)w * h; ++i) out[i] = (uint8_t)(mt_next(&m) & 0xFFu);
}

void stk_synth_random_mask(int w, int h, uint32_t seed, int percent, uint8_t* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (size_t i = 0; i < (size_t)w * h; ++i)
        out[i] = (mt_next(&m) % 100u) < (uint32_t)percent ? 1 : 0;
}

void stk_synth_random_sparse(int w, int h, uint32_t seed, int percent, int dmax, int16_t* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        out[i] = -1;
        if ((mt_next(&m) % 100u) < (uint32_t)percent)
            out[i] = (int16_t)(mt_next(&m) % (uint32_t)(dmax + 1));
    }
}

/* left(x) = wide(x), right(x) = wide(x + shift) */
static void split_wide(const uint8_t* wide, int ww, int w, int h, int shift, uint8_t* l,
                       uint8_t* r) {
    for (int y = 0; y < h; ++y) {
        memcpy(l + (size_t)y * w * 3, wide + (size_t)y * ww * 3, (size_t)w * 3);
        memcpy(r + (size_t)y * w * 3, wide + ((size_t)y * ww + shift) * 3, (size_t)w * 3);
    }
}

static void grey_rect(uint8_t* im, int ww, mt_t* m, int x0, int y0, int x1, int y1, int base,
                      int spread) {
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
            const uint8_t v = (uint8_t)(base + (int)(mt_next(m) % (uint32_t)spread));
            uint8_t* p = im + ((size_t)y * ww + x) * 3;
            p[0] = p[1] = p[2] = v;
        }
}

void stk_synth_translated_noise(int w, int h, int shift, uint32_t seed, uint8_t* l, uint8_t* r) {
    const int ww = w + shift;
    uint8_t* wide = (uint8_t*)malloc((size_t)ww * h * 3 + 1);
    stk_synth_random_rgb(ww, h, seed, wide);
    split_wide(wide, ww, w, h, shift, l, r);
    free(wide);
}

void stk_synth_rectangle_scene(int w, int h, int shift, uint32_t seed, uint8_t* l, uint8_t* r) {
    const int ww = w + shift;
    uint8_t* wide = (uint8_t*)calloc((size_t)ww * h * 3 + 1, 1);
    mt_t m;
    mt_seed(&m, seed);
    grey_rect(wide, ww, &m, 0, 0, ww, h, 20, 50);
    grey_rect(wide, ww, &m, w * 2 / 10, h * 2 / 10, w * 4 / 10, h * 5 / 10, 150, 70);
    grey_rect(wide, ww, &m, w * 6 / 10, h * 55 / 100, w * 9 / 10, h * 85 / 100, 150, 70);
    split_wide(wide, ww, w, h, shift, l, r);
    free(wide);
}

void stk_synth_bench_frame(int w, int h, uint32_t seed, uint8_t* l, uint8_t* r) {
    const int shift = 5, ww = w + shift, cell = 96;
    const int bases[4] = {60, 110, 160, 210};
    uint8_t* wide = (uint8_t*)calloc((size_t)ww * h * 3 + 1, 1);
    mt_t m;
    mt_seed(&m, seed);
    grey_rect(wide, ww, &m, 0, 0, ww, h, 8, 40);
    int band = 0;
    for (int gy = 12; gy + cell < h - 12; gy += cell + 14)
        for (int gx = 12; gx + cell < w - 12; gx += cell + 14) {
            const int ix = (int)(mt_next(&m) % 24u);
            const int iy = (int)(mt_next(&m) % 24u);
            grey_rect(wide, ww, &m, gx + ix, gy + iy, gx + cell - 4, gy + cell - 4,
                      bases[band % 4], 36);
            ++band;
        }
    split_wide(wide, ww, w, h, shift, l, r);
    free(wide);
}

typedef struct {
    int w, h, x0, y0, d, base, idx;
} leaf_t;

static int leaf_cmp(const void* a, const void* b) {
    const leaf_t *p = (const leaf_t*)a, *q = (const leaf_t*)b;
    if (p->d != q->d) return p->d < q->d ? -1 : 1;
    return p->idx < q->idx ? -1 : (p->idx > q->idx); /* stable */
}

/* G2 "dead leaves": rects = round(W*H/281.25) grey
 * rectangles of side U[4,30] and disparity U[0,D], painted far to near over a
 * dark noise background at disparity 0; the right view shifts each rectangle
 * left by its disparity.  Seed = 2001 + frame index. */
void stk_synth_dead_leaves(int w, int h, int max_disparity, uint32_t seed, uint8_t* l,
                           uint8_t* r) {
    const int min_side = 4, max_side = 30, noise = 6;
    const long nrect = (long)((double)w * h / 281.25 + 0.5);
    leaf_t* lv = (leaf_t*)malloc(sizeof(leaf_t) * (size_t)(nrect + 1));
    mt_t m;
    mt_seed(&m, seed);
    for (long i = 0; i < nrect; ++i) {
        leaf_t* p = &lv[i];
        p->w = min_side + (int)(mt_next(&m) % (uint32_t)(max_side - min_side + 1));
        p->h = min_side + (int)(mt_next(&m) % (uint32_t)(max_side - min_side + 1));
        p->x0 = (int)(mt_next(&m) % (uint32_t)w) - p->w / 2;
        p->y0 = (int)(mt_next(&m) % (uint32_t)h) - p->h / 2;
        p->d = (int)(mt_next(&m) % (uint32_t)(max_disparity + 1));
        p->base = 16 + (int)(mt_next(&m) % 200u);
        p->idx = (int)i;
    }
    qsort(lv, (size_t)nrect, sizeof(leaf_t), leaf_cmp);
    const size_t n = (size_t)w * h;
    for (size_t p = 0; p < n; ++p) {
        const uint8_t v = (uint8_t)(8 + mt_next(&m) % (uint32_t)(noise + 1));
        l[3 * p] = l[3 * p + 1] = l[3 * p + 2] = v;
        r[3 * p] = r[3 * p + 1] = r[3 * p + 2] = v;
    }
    for (long i = 0; i < nrect; ++i) {
        const leaf_t* p = &lv[i];
        const int ya = p->y0 < 0 ? 0 : p->y0, yb = p->y0 + p->h < h ? p->y0 + p->h : h;
        const int xa = p->x0 < 0 ? 0 : p->x0, xb = p->x0 + p->w < w ? p->x0 + p->w : w;
        for (int y = ya; y < yb; ++y)
            for (int x = xa; x < xb; ++x) {
                int v = p->base + (int)(mt_next(&m) % (uint32_t)(noise + 1));
                if (v > 255) v = 255;
                uint8_t* pl = l + ((size_t)y * w + x) * 3;
                pl[0] = pl[1] = pl[2] = (uint8_t)v;
                if (x - p->d >= 0) {
                    uint8_t* pr = r + ((size_t)y * w + (x - p->d)) * 3;
                    pr[0] = pr[1] = pr[2] = (uint8_t)v;
                }
            }
    }
    free(lv);
}
