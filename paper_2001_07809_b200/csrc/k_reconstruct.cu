// K6 fill_rows + K7 peek_cols -- dense reconstruction from the sparse map
// (reference: reconstruct.cpp:11-109, the paper's Algorithms 1 and 2).
//
// K6: one CTA per row; every thread owns a contiguous chunk (16 pixels in
//     registers when W % 16 == 0, else a shared-memory row), and block scans
//     give each chunk the nearest known on either side.  A run of unknowns
//     between consecutive knowns of equal disparity is filled; knowns never
//     change (reconstruct.cpp:11-33).
// K7: one CTA per 16 columns x 64 row segments.  One pass summarises each
//     segment (known count, first two / last two knowns); warp-level scans
//     derive, per segment, the nearest known above/below and, per column,
//     the first two / last two knowns; a second pass walks the segment again
//     and resolves each unknown with peek_estimate (reconstruct.cpp:40-46)
//     on the snapshot:
//       0 knowns -> stays unknown, 1 known -> copy,
//       above & below -> est(above, below),
//       nothing above -> est(first two), nothing below -> est(last two).
#include <cstdlib>

#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int kFillThreads = 256;

__device__ __forceinline__ int16_t peek_estimate(int a, int b, int thr) {
    const int r = a >= b ? a - b : b - a;
    if (r > thr) return (int16_t)(a < b ? a : b);
    return (int16_t)((a + b) / 2);
}

// ------------------------------------------------------------------ K6 ----
__global__ void __launch_bounds__(kFillThreads) k_fill_rows(Frame f, const int16_t* __restrict__ in,
                                                            int16_t* __restrict__ out) {
    extern __shared__ int16_t row[];
    __shared__ uint32_t wl[kFillThreads / 32], wf[kFillThreads / 32];
    const int W = f.W, y = blockIdx.x, tid = threadIdx.x;
    const int16_t* src = in + (size_t)y * W;
    for (int x = tid; x < W; x += kFillThreads) row[x] = src[x];
    __syncthreads();
    const int ch = (W + kFillThreads - 1) / kFillThreads;
    const int a = min(W, tid * ch), b = min(W, a + ch);
    // last known in my chunk as ((x+1)<<16 | d), first known as (x<<16 | d)
    uint32_t klast = 0, kfirst = 0xffffffffu;
    for (int x = a; x < b; ++x) {
        const int16_t d = row[x];
        if (d >= 0) {
            klast = ((uint32_t)(x + 1) << 16) | (uint16_t)d;
            if (kfirst == 0xffffffffu) kfirst = ((uint32_t)x << 16) | (uint16_t)d;
        }
    }
    // exclusive max-scan (prev) and exclusive reverse min-scan (next)
    const int lane = tid & 31, wid = tid >> 5;
    uint32_t incl_l = klast;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl_l, o);
        if (lane >= o) incl_l = max(incl_l, v);
    }
    uint32_t incl_f = kfirst;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, incl_f, o);
        if (lane + o < 32) incl_f = min(incl_f, v);
    }
    if (lane == 31) wl[wid] = incl_l;
    if (lane == 0) wf[wid] = incl_f;
    __syncthreads();
    uint32_t prev = __shfl_up_sync(0xffffffffu, incl_l, 1);
    if (lane == 0) prev = 0;
    for (int i = 0; i < wid; ++i) prev = max(prev, wl[i]);
    uint32_t next = __shfl_down_sync(0xffffffffu, incl_f, 1);
    if (lane == 31) next = 0xffffffffu;
    for (int i = wid + 1; i < kFillThreads / 32; ++i) next = min(next, wf[i]);
    // walk my chunk
    bool have_prev = prev != 0;
    int pd = have_prev ? (int)(prev & 0xffffu) : -1;
    int rs = -1;
    for (int x = a; x < b; ++x) {
        const int16_t d = row[x];
        if (d >= 0) {
            if (rs >= 0 && have_prev && pd == d)
                for (int q = rs; q < x; ++q) row[q] = d;
            rs = -1;
            have_prev = true;
            pd = d;
        } else if (rs < 0) {
            rs = x;
        }
    }
    if (rs >= 0 && have_prev && next != 0xffffffffu && (int)(next & 0xffffu) == pd)
        for (int q = rs; q < b; ++q) row[q] = (int16_t)pd;
    __syncthreads();
    int16_t* dst = out + (size_t)y * W;
    for (int x = tid; x < W; x += kFillThreads) dst[x] = row[x];
}

// K6 v3 (W % 16 == 0): CTA per row, 16 pixels per thread in registers
// (2 x 16-byte loads / stores), value-only scans: a pixel is filled iff its nearest known
// on the left and on the right both exist and are equal, so the chunk only
// publishes its last / first known value (-1 = none) and the block scans use
// "latest / earliest known" operators -- no positions, no int16 arrays.
__global__ void __launch_bounds__(1024) k_fill_rows16v(Frame f, const int16_t* __restrict__ in,
                                                       int16_t* __restrict__ out) {
    __shared__ int wl[32], wf[32];
    const unsigned full = 0xffffffffu;
    const int W = f.W, y = blockIdx.x, tid = threadIdx.x;
    const bool act = tid < W / 16;
    const int x0 = tid * 16;
    uint32_t w[8];
    {
        uint4 a = make_uint4(full, full, full, full), b = a;
        if (act) {
            const uint4* src = reinterpret_cast<const uint4*>(in + (size_t)y * W + x0);
            a = __ldcs(src);
            b = __ldcs(src + 1);
        }
        w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
    }
    int v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[2 * i] = (int)(w[i] << 16) >> 16;
        v[2 * i + 1] = (int)w[i] >> 16;
    }
    int lastv = -1, firstv = -1;
#pragma unroll
    for (int i = 0; i < 16; ++i) lastv = v[i] >= 0 ? v[i] : lastv;
#pragma unroll
    for (int i = 15; i >= 0; --i) firstv = v[i] >= 0 ? v[i] : firstv;
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    int inc = lastv;  // latest known over lanes <= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(full, inc, o);
        if (lane >= o && inc < 0) inc = t;
    }
    int sinc = firstv;  // earliest known over lanes >= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_down_sync(full, sinc, o);
        if (lane + o < 32 && sinc < 0) sinc = t;
    }
    if (lane == 31) wl[wid] = inc;
    if (lane == 0) wf[wid] = sinc;
    __syncthreads();
    int pd = __shfl_up_sync(full, inc, 1);
    if (lane == 0) pd = -1;
    if (pd < 0)
        for (int i = wid - 1; i >= 0 && pd < 0; --i) pd = wl[i];
    int nd = __shfl_down_sync(full, sinc, 1);
    if (lane == 31) nd = -1;
    if (nd < 0)
        for (int i = wid + 1; i < nw && nd < 0; ++i) nd = wf[i];
    if (!act) return;
    // right context of each pixel: the nearest known at or right of it
    int r[16];
#pragma unroll
    for (int i = 15; i >= 0; --i) {
        r[i] = nd;
        nd = v[i] >= 0 ? v[i] : nd;
    }
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        // unknown: filled iff nearest left == nearest right (both -1 -> stays -1)
        const int val = v[i] >= 0 ? v[i] : (pd == r[i] ? pd : -1);
        pd = v[i] >= 0 ? v[i] : pd;
        if (i & 1) o[i >> 1] |= (uint32_t)val << 16;
        else o[i >> 1] = (uint32_t)val & 0xffffu;
    }
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)y * W + x0);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

// ------------------------------------------------------------------ K7 ----
constexpr int PC = 16;  // columns per CTA (a warp = 16 columns x 2 segments)
constexpr int PS = 64;  // row segments per column
constexpr int PB = 12;  // rows loaded per batch (independent loads in flight)

struct SegSum {
    int count;     // knowns in the segment
    int16_t f1, f2;  // first two knowns (top-down), -1 if absent
    int16_t l1, l2;  // last known, second last, -1 if absent
};

// K7 v2: the same segments, branch-free.  Pass 1 (top-down) builds the
// segment summary and stores, per pixel, the nearest known above it inside the
// segment (or -1) into `out` as scratch; after the cross-segment context
// (phase 2) pass 2 walks the segment bottom-up carrying the nearest known
// below and resolves every pixel with selects.
__global__ void __launch_bounds__(PC * PS) k_peek_cols2(Frame f, const int16_t* __restrict__ in,
                                                        int16_t* __restrict__ out) {
    __shared__ SegSum seg[PS][PC];
    __shared__ int16_t ctx_ab[PS][PC], ctx_bl[PS][PC];  // nearest known above / below a segment
    __shared__ int col_total[PC], col_top[PC], col_bot[PC];
    __shared__ unsigned long long red[PC * PS / 32];
    const int W = f.W, H = f.H, thr = f.thr;
    const int cx = threadIdx.x % PC, s = threadIdx.x / PC;
    const int x = blockIdx.x * PC + cx;
    const int sr = (H + PS - 1) / PS;
    const int ya = min(H, s * sr), yb = min(H, ya + sr);
    const bool col = x < W;
    // pass 1 (top-down): segment summary; nearest known above inside the
    // segment (or -1) parked in `out`
    SegSum m{0, -1, -1, -1, -1};
    if (col) {
        int cur = -1;
        const int16_t* ip = in + (size_t)ya * W + x;
        int16_t* op = out + (size_t)ya * W + x;
        for (int yy = ya; yy < yb; yy += PB, ip += (size_t)PB * W, op += (size_t)PB * W) {
            const int n = min(PB, yb - yy);
            int16_t v[PB];
#pragma unroll
            for (int k = 0; k < PB; ++k) v[k] = k < n ? __ldg(ip + (size_t)k * W) : (int16_t)-1;
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                if (k < n) op[(size_t)k * W] = (int16_t)cur;
                const int d = v[k];
                const bool kn = d >= 0;
                m.f2 = (kn && m.count == 1) ? (int16_t)d : m.f2;
                m.f1 = (kn && m.count == 0) ? (int16_t)d : m.f1;
                m.l2 = kn ? m.l1 : m.l2;
                m.l1 = kn ? (int16_t)d : m.l1;
                m.count += kn;
                cur = kn ? d : cur;
            }
        }
    }
    seg[s][cx] = m;
    __syncthreads();
    // phase 2: one thread per column scans the segments once
    if (s == 0) {
        int total = 0, last = -1;
        int cf1 = -1, cf2 = -1;
        for (int i = 0; i < PS; ++i) {
            const SegSum g = seg[i][cx];
            ctx_ab[i][cx] = (int16_t)last;
            if (g.count) {
                last = g.l1;
                if (cf1 < 0) {
                    cf1 = g.f1;
                    if (g.count > 1) cf2 = g.f2;
                } else if (cf2 < 0) {
                    cf2 = g.f1;
                }
            }
            total += g.count;
        }
        int first = -1, cl1 = -1, cl2 = -1;
        for (int i = PS - 1; i >= 0; --i) {
            const SegSum g = seg[i][cx];
            ctx_bl[i][cx] = (int16_t)first;
            if (g.count) {
                first = g.f1;
                if (cl1 < 0) {
                    cl1 = g.l1;
                    if (g.count > 1) cl2 = g.l2;
                } else if (cl2 < 0) {
                    cl2 = g.l1;
                }
            }
        }
        col_total[cx] = total;
        col_top[cx] = total >= 2 ? peek_estimate(cf1, cf2, thr) : -1;
        col_bot[cx] = total >= 2 ? peek_estimate(cl2, cl1, thr) : -1;
    }
    __syncthreads();
    const int total = col_total[cx], est_top = col_top[cx], est_bot = col_bot[cx];
    const int above = ctx_ab[s][cx];
    // pass 2 (bottom-up): nearest known below carried, every pixel resolved
    unsigned long long known = 0;
    if (col) {
        int nb = ctx_bl[s][cx];
        for (int yy = yb - 1; yy >= ya; yy -= PB) {
            const int n = min(PB, yy - ya + 1);
            int16_t v[PB], a[PB];
            const int16_t* ip = in + (size_t)yy * W + x;
            int16_t* op = out + (size_t)yy * W + x;
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                v[k] = k < n ? __ldg(ip - (size_t)k * W) : (int16_t)-1;
                a[k] = k < n ? op[-(long long)k * W] : (int16_t)-1;
            }
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                if (k >= n) break;
                const int d = v[k];
                const int ab = a[k] >= 0 ? a[k] : above;  // nearest known above
                int r;
                if (d >= 0) r = d;
                else if (total == 0) r = -1;
                else if (total == 1) r = ab >= 0 ? ab : nb;
                else if (ab >= 0 && nb >= 0) r = peek_estimate(ab, nb, thr);
                else r = ab < 0 ? est_top : est_bot;
                op[-(long long)k * W] = (int16_t)r;
                known += r >= 0;
                nb = d >= 0 ? d : nb;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = known;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < PC * PS / 32; ++i) t += red[i];
        if (t) atomicAdd(&f.sc->known, t);
    }
}

// K7 helpers for the two-columns-per-thread kernel (int16 pairs in 32-bit
// loads/stores: a warp's 8 column pairs x 4 segments move 32 contiguous bytes
// per row each).
#ifndef STK_P4B
#define STK_P4B 12
#endif
constexpr int P4B = STK_P4B;  // rows per load batch (4K peek: 8 rows 29 us, 12: 27.5, 16: 30.6)

__device__ __forceinline__ uint32_t pack2(int a, int b) { return (uint32_t)(uint16_t)a | (uint32_t)b << 16; }
__device__ __forceinline__ int lo16(uint32_t v) { return (int16_t)(v & 0xffffu); }
__device__ __forceinline__ int hi16s(uint32_t v) { return (int16_t)(v >> 16); }

// K7 v5 (even W; k_peek_cols2 otherwise): 16 columns x 64 row segments per
// CTA, two adjacent columns per thread, lean passes:
//   pass 1 (bottom-up): the nearest known strictly below within the segment
//     goes to `out` as scratch, and the segment summary (count, first two,
//     last two knowns) to shared memory;
//   phase 2: warp w = column w; lanes hold 2 segments each and warp shuffles
//     give every segment its nearest known above / below (ordered scans) and
//     the column its first two / last two knowns (ordered tree reductions) --
//     no serial per-column loop;
//   pass 2 (top-down): each pixel resolved from (input, nearest above carried
//     in a register, nearest below from the scratch or the segment context).
constexpr int P5C = 8;   // column pairs per CTA (16 columns)
constexpr int P5S = 64;  // row segments per column (= 2 x 32 lanes in phase 2)

// Branch-free (selects only): the cases of reconstruct.cpp:57-106 for one
// pixel given its nearest known above (a) and below (b), -1 = none.  The
// column's total is folded into et / eb by the caller: total == 0 -> both -1,
// total == 1 -> a or b is the single known, so "a < 0 ? b : a" covers it.
__device__ __forceinline__ int peek_resolve(int d, int a, int b, int single, int et, int eb, int thr) {
    const int r = a >= b ? a - b : b - a;
    const int est = r > thr ? min(a, b) : (a + b) >> 1;
    const int edge = a < 0 ? et : eb;
    const int two = (a >= 0 && b >= 0) ? est : edge;
    const int one = a >= 0 ? a : b;
    const int u = single ? one : two;
    return d >= 0 ? d : u;
}

__global__ void __launch_bounds__(P5C * P5S, 2) k_peek_cols5(Frame f, const int16_t* __restrict__ in,
                                                          int16_t* __restrict__ out) {
    __shared__ int s_cnt[P5S][2 * P5C];
    __shared__ uint32_t s_first[P5S][2 * P5C];  // f1 | f2 << 16 (int16 each, -1 = none)
    __shared__ uint32_t s_last[P5S][2 * P5C];   // l1 | l2 << 16 (last, second last)
    __shared__ int16_t ctx_ab[P5S][2 * P5C], ctx_bl[P5S][2 * P5C];
    __shared__ int col_total[2 * P5C], col_top[2 * P5C], col_bot[2 * P5C];
    __shared__ unsigned long long red[P5C * P5S / 32];
    const int W = f.W, H = f.H, thr = f.thr;
    const int cp = threadIdx.x % P5C, s = threadIdx.x / P5C;
    const int x = 2 * (blockIdx.x * P5C + cp);  // W even
    const int sr = (H + P5S - 1) / P5S;
    const int ya = min(H, s * sr), yb = min(H, ya + sr);
    const bool col = x < W;
    const uint32_t* __restrict__ in2 = reinterpret_cast<const uint32_t*>(in);
    uint32_t* __restrict__ out2 = reinterpret_cast<uint32_t*>(out);
    const size_t W2 = (size_t)W / 2;
    // ---- pass 1 (bottom-up)
    int n0 = 0, n1 = 0, b0 = -1, b1 = -1;
    int f10 = -1, f20 = -1, l10 = -1, l20 = -1, f11 = -1, f21 = -1, l11 = -1, l21 = -1;
    if (col) {
        const uint32_t* ip = in2 + x / 2 + (size_t)(yb - 1) * W2;
        uint32_t* op = out2 + x / 2 + (size_t)(yb - 1) * W2;
        auto row = [&](uint32_t v, uint32_t* dst) {
            *dst = pack2(b0, b1);
            const int d0 = lo16(v), d1 = hi16s(v);
            if (d0 >= 0) {
                l20 = n0 == 1 ? d0 : l20;
                l10 = n0 == 0 ? d0 : l10;
                f20 = f10;
                f10 = d0;
                b0 = d0;
                ++n0;
            }
            if (d1 >= 0) {
                l21 = n1 == 1 ? d1 : l21;
                l11 = n1 == 0 ? d1 : l11;
                f21 = f11;
                f11 = d1;
                b1 = d1;
                ++n1;
            }
        };
        int y = yb - 1;
        for (; y - P4B + 1 >= ya; y -= P4B, ip -= P4B * W2, op -= P4B * W2) {
            uint32_t v[P4B];
#pragma unroll
            for (int k = 0; k < P4B; ++k) v[k] = __ldg(ip - k * W2);
#pragma unroll
            for (int k = 0; k < P4B; ++k) row(v[k], op - k * W2);
        }
        for (; y >= ya; --y, ip -= W2, op -= W2) row(__ldg(ip), op);
    }
    s_cnt[s][2 * cp] = n0;
    s_cnt[s][2 * cp + 1] = n1;
    s_first[s][2 * cp] = pack2(f10, f20);
    s_first[s][2 * cp + 1] = pack2(f11, f21);
    s_last[s][2 * cp] = pack2(l10, l20);
    s_last[s][2 * cp + 1] = pack2(l11, l21);
    __syncthreads();
    // ---- phase 2: warp = column, lane = segments (2 lane, 2 lane + 1)
    {
        const unsigned full = 0xffffffffu;
        const int cx = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int i0 = 2 * lane, i1 = i0 + 1;
        const int c0 = s_cnt[i0][cx], c1 = s_cnt[i1][cx];
        const uint32_t F0 = s_first[i0][cx], F1 = s_first[i1][cx];
        const uint32_t L0 = s_last[i0][cx], L1 = s_last[i1][cx];
        // nearest known above each segment: "latest known" exclusive scan
        int inc = c1 ? lo16(L1) : (c0 ? lo16(L0) : -1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(full, inc, o);
            if (lane >= o && inc < 0) inc = t;
        }
        int ex = __shfl_up_sync(full, inc, 1);
        if (lane == 0) ex = -1;
        ctx_ab[i0][cx] = (int16_t)ex;
        ctx_ab[i1][cx] = (int16_t)(c0 ? lo16(L0) : ex);
        // nearest known below each segment: "earliest known" suffix scan
        int sinc = c0 ? lo16(F0) : (c1 ? lo16(F1) : -1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_down_sync(full, sinc, o);
            if (lane + o < 32 && sinc < 0) sinc = t;
        }
        int sx = __shfl_down_sync(full, sinc, 1);
        if (lane == 31) sx = -1;
        ctx_bl[i1][cx] = (int16_t)sx;
        ctx_bl[i0][cx] = (int16_t)(c1 ? lo16(F1) : sx);
        const int total = __reduce_add_sync(full, c0 + c1);
        // first two knowns of the column: ordered combine of (k1, k2)
        auto comb_first = [](int a1, int a2, int b1, int& r1, int& r2) {
            if (a2 >= 0) { r1 = a1; r2 = a2; }
            else if (a1 >= 0) { r1 = a1; r2 = b1; }
            else { r1 = b1; r2 = -2; }  // -2: take b's second below
        };
        int k1, k2;
        {
            int r1, r2;
            comb_first(lo16(F0), hi16s(F0), lo16(F1), r1, r2);
            k1 = r1;
            k2 = r2 == -2 ? hi16s(F1) : r2;
        }
        // last two: (m1 = last, m2 = second last), ordered combine, later wins
        int m1, m2;
        if (hi16s(L1) >= 0) { m1 = lo16(L1); m2 = hi16s(L1); }
        else if (lo16(L1) >= 0) { m1 = lo16(L1); m2 = lo16(L0); }
        else { m1 = lo16(L0); m2 = hi16s(L0); }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ok1 = __shfl_down_sync(full, k1, o), ok2 = __shfl_down_sync(full, k2, o);
            const int om1 = __shfl_down_sync(full, m1, o), om2 = __shfl_down_sync(full, m2, o);
            if ((lane & (2 * o - 1)) == 0 && lane + o < 32) {
                // this lane's range precedes the other's
                if (k2 < 0) {
                    if (k1 >= 0) k2 = ok1;
                    else { k1 = ok1; k2 = ok2; }
                }
                if (om2 >= 0) { m1 = om1; m2 = om2; }
                else if (om1 >= 0) { m2 = m1; m1 = om1; }
            }
        }
        if (lane == 0) {
            col_total[cx] = total;
            col_top[cx] = total >= 2 ? peek_estimate(k1, k2, thr) : -1;
            col_bot[cx] = total >= 2 ? peek_estimate(m2, m1, thr) : -1;
        }
    }
    __syncthreads();
    // ---- pass 2 (top-down)
    unsigned long long known = 0;
    if (col) {
        const int t0 = col_total[2 * cp], t1 = col_total[2 * cp + 1];
        // total 0: every estimate is -1; total 1: the single known is a or b
        const int sg0 = t0 == 1, sg1 = t1 == 1;
        const int et0 = t0 ? col_top[2 * cp] : -1, et1 = t1 ? col_top[2 * cp + 1] : -1;
        const int eb0 = t0 ? col_bot[2 * cp] : -1, eb1 = t1 ? col_bot[2 * cp + 1] : -1;
        int a0 = ctx_ab[s][2 * cp], a1 = ctx_ab[s][2 * cp + 1];
        const int bl0 = ctx_bl[s][2 * cp], bl1 = ctx_bl[s][2 * cp + 1];
        const uint32_t* ip = in2 + x / 2 + (size_t)ya * W2;
        uint32_t* op = out2 + x / 2 + (size_t)ya * W2;
        auto row = [&](uint32_t v, uint32_t bw, uint32_t* dst) {
            const int d0 = lo16(v), d1 = hi16s(v);
            const int s0 = lo16(bw), s1 = hi16s(bw);
            const int r0 = peek_resolve(d0, a0, s0 >= 0 ? s0 : bl0, sg0, et0, eb0, thr);
            const int r1 = peek_resolve(d1, a1, s1 >= 0 ? s1 : bl1, sg1, et1, eb1, thr);
            a0 = d0 >= 0 ? d0 : a0;
            a1 = d1 >= 0 ? d1 : a1;
            *dst = pack2(r0, r1);
            known += (r0 >= 0) + (r1 >= 0);
        };
        // batches: all loads of P4B rows (input and scratch) issue before the
        // stores (the scratch loads would otherwise wait behind them)
        int y = ya;
        for (; y + P4B <= yb; y += P4B, ip += P4B * W2, op += P4B * W2) {
            uint32_t v[P4B], bw[P4B];
#pragma unroll
            for (int k = 0; k < P4B; ++k) {
                v[k] = __ldg(ip + k * W2);
                bw[k] = op[k * W2];
            }
#pragma unroll
            for (int k = 0; k < P4B; ++k) row(v[k], bw[k], op + k * W2);
        }
        for (; y < yb; ++y, ip += W2, op += W2) row(__ldg(ip), *op, op);
    }
    for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = known;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < P5C * P5S / 32; ++i) t += red[i];
        if (t) atomicAdd(&f.sc->known, t);
    }
}

// int16x2 lane helpers for K7 v6: sign masks, per-lane add / min / max
// (__byte_perm drops bit 3 of the selector nibbles: the sign-replicating
// selector 0xbb99 needs prmt itself)
__device__ __forceinline__ uint32_t sgn2(uint32_t v) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xbb99;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint32_t vadd2(uint32_t a, uint32_t b) { return __vadd2(a, b); }
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vmins2(a, b); }
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }

// K7 v6: K7 v5 with both columns of a thread in int16x2 lanes (PRMT sign
// masks, LOP3 selects, VIADD/VIMNMX.16x2): half the instructions per row.
// SMEM: the nearest-below scratch lives in shared memory ([H][P5C] u32, the
// CTA's 16 columns) instead of in `out` (3 global passes instead of 5)
template <bool SMEM>
__global__ void __launch_bounds__(P5C * P5S, 2) k_peek_cols6(Frame f, const int16_t* __restrict__ in,
                                                          int16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t scr[];
    __shared__ int s_cnt[P5S][2 * P5C];
    __shared__ uint32_t s_first[P5S][2 * P5C];  // f1 | f2 << 16 (int16 each, -1 = none)
    __shared__ uint32_t s_last[P5S][2 * P5C];   // l1 | l2 << 16 (last, second last)
    __shared__ int16_t ctx_ab[P5S][2 * P5C], ctx_bl[P5S][2 * P5C];
    __shared__ int col_total[2 * P5C], col_top[2 * P5C], col_bot[2 * P5C];
    __shared__ unsigned long long red[P5C * P5S / 32];
    const int W = f.W, H = f.H, thr = f.thr;
    const int cp = threadIdx.x % P5C, s = threadIdx.x / P5C;
    const int x = 2 * (blockIdx.x * P5C + cp);  // W even
    const int sr = (H + P5S - 1) / P5S;
    const int ya = min(H, s * sr), yb = min(H, ya + sr);
    const bool col = x < W;
    const uint32_t* __restrict__ in2 = reinterpret_cast<const uint32_t*>(in);
    uint32_t* __restrict__ out2 = reinterpret_cast<uint32_t*>(out);
    const size_t W2 = (size_t)W / 2;
    // ---- pass 1 (bottom-up), both columns in int16x2 lanes: lane masks by
    // sign replication (PRMT 0xbb99: 0xffff where negative), selects by LOP3.
    //   f1 / f2: nearest / second nearest known going up (the segment's first
    //   two from the top once the walk ends; f1 is also "nearest known
    //   below" for the rows above), l1 / l2: the first two met (the
    //   segment's last two), n2: known counts.
    uint32_t f1 = 0xffffffffu, f2 = 0xffffffffu, l1 = 0xffffffffu, l2 = 0xffffffffu, n2 = 0;
    if (col) {
        const uint32_t* ip = in2 + x / 2 + (size_t)(yb - 1) * W2;
        const size_t OS = SMEM ? (size_t)P5C : W2;  // scratch row stride
        uint32_t* op = SMEM ? scr + cp + (size_t)(yb - 1) * P5C : out2 + x / 2 + (size_t)(yb - 1) * W2;
        auto row = [&](uint32_t v, uint32_t* dst) {
            *dst = f1;
            const uint32_t md = sgn2(v);  // unknown lanes
            const uint32_t m2 = ~md & ~sgn2(l1) & sgn2(l2);
            l2 = (v & m2) | (l2 & ~m2);
            const uint32_t m1 = ~md & sgn2(l1);
            l1 = (v & m1) | (l1 & ~m1);
            f2 = (f2 & md) | (f1 & ~md);
            f1 = (f1 & md) | (v & ~md);
            n2 += ~md & 0x00010001u;
        };
        int y = yb - 1;
        for (; y - P4B + 1 >= ya; y -= P4B, ip -= P4B * W2, op -= P4B * OS) {
            uint32_t v[P4B];
#pragma unroll
            for (int k = 0; k < P4B; ++k) v[k] = __ldg(ip - k * W2);
#pragma unroll
            for (int k = 0; k < P4B; ++k) row(v[k], op - k * OS);
        }
        for (; y >= ya; --y, ip -= W2, op -= OS) row(__ldg(ip), op);
    }
    s_cnt[s][2 * cp] = (int)(n2 & 0xffffu);
    s_cnt[s][2 * cp + 1] = (int)(n2 >> 16);
    s_first[s][2 * cp] = pack2(lo16(f1), lo16(f2));
    s_first[s][2 * cp + 1] = pack2(hi16s(f1), hi16s(f2));
    s_last[s][2 * cp] = pack2(lo16(l1), lo16(l2));
    s_last[s][2 * cp + 1] = pack2(hi16s(l1), hi16s(l2));
    __syncthreads();
    // ---- phase 2: warp = column, lane = segments (2 lane, 2 lane + 1)
    {
        const unsigned full = 0xffffffffu;
        const int cx = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int i0 = 2 * lane, i1 = i0 + 1;
        const int c0 = s_cnt[i0][cx], c1 = s_cnt[i1][cx];
        const uint32_t F0 = s_first[i0][cx], F1 = s_first[i1][cx];
        const uint32_t L0 = s_last[i0][cx], L1 = s_last[i1][cx];
        // nearest known above each segment: "latest known" exclusive scan
        int inc = c1 ? lo16(L1) : (c0 ? lo16(L0) : -1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(full, inc, o);
            if (lane >= o && inc < 0) inc = t;
        }
        int ex = __shfl_up_sync(full, inc, 1);
        if (lane == 0) ex = -1;
        ctx_ab[i0][cx] = (int16_t)ex;
        ctx_ab[i1][cx] = (int16_t)(c0 ? lo16(L0) : ex);
        // nearest known below each segment: "earliest known" suffix scan
        int sinc = c0 ? lo16(F0) : (c1 ? lo16(F1) : -1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_down_sync(full, sinc, o);
            if (lane + o < 32 && sinc < 0) sinc = t;
        }
        int sx = __shfl_down_sync(full, sinc, 1);
        if (lane == 31) sx = -1;
        ctx_bl[i1][cx] = (int16_t)sx;
        ctx_bl[i0][cx] = (int16_t)(c1 ? lo16(F1) : sx);
        const int total = __reduce_add_sync(full, c0 + c1);
        // first two knowns of the column: ordered combine of (k1, k2)
        auto comb_first = [](int a1, int a2, int b1, int& r1, int& r2) {
            if (a2 >= 0) { r1 = a1; r2 = a2; }
            else if (a1 >= 0) { r1 = a1; r2 = b1; }
            else { r1 = b1; r2 = -2; }  // -2: take b's second below
        };
        int k1, k2;
        {
            int r1, r2;
            comb_first(lo16(F0), hi16s(F0), lo16(F1), r1, r2);
            k1 = r1;
            k2 = r2 == -2 ? hi16s(F1) : r2;
        }
        // last two: (m1 = last, m2 = second last), ordered combine, later wins
        int m1, m2;
        if (hi16s(L1) >= 0) { m1 = lo16(L1); m2 = hi16s(L1); }
        else if (lo16(L1) >= 0) { m1 = lo16(L1); m2 = lo16(L0); }
        else { m1 = lo16(L0); m2 = hi16s(L0); }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ok1 = __shfl_down_sync(full, k1, o), ok2 = __shfl_down_sync(full, k2, o);
            const int om1 = __shfl_down_sync(full, m1, o), om2 = __shfl_down_sync(full, m2, o);
            if ((lane & (2 * o - 1)) == 0 && lane + o < 32) {
                // this lane's range precedes the other's
                if (k2 < 0) {
                    if (k1 >= 0) k2 = ok1;
                    else { k1 = ok1; k2 = ok2; }
                }
                if (om2 >= 0) { m1 = om1; m2 = om2; }
                else if (om1 >= 0) { m2 = m1; m1 = om1; }
            }
        }
        if (lane == 0) {
            col_total[cx] = total;
            col_top[cx] = total >= 2 ? peek_estimate(k1, k2, thr) : -1;
            col_bot[cx] = total >= 2 ? peek_estimate(m2, m1, thr) : -1;
        }
    }
    __syncthreads();
    // ---- pass 2 (top-down), int16x2 lanes as pass 1 (peek_resolve per lane)
    unsigned long long known = 0;
    if (col) {
        const int t0 = col_total[2 * cp], t1 = col_total[2 * cp + 1];
        // total 0: every estimate is -1; total 1: the single known is a or b
        const uint32_t sg = (t0 == 1 ? 0x0000ffffu : 0u) | (t1 == 1 ? 0xffff0000u : 0u);
        const uint32_t et = pack2(t0 ? col_top[2 * cp] : -1, t1 ? col_top[2 * cp + 1] : -1);
        const uint32_t eb = pack2(t0 ? col_bot[2 * cp] : -1, t1 ? col_bot[2 * cp + 1] : -1);
        uint32_t a = pack2(ctx_ab[s][2 * cp], ctx_ab[s][2 * cp + 1]);
        const uint32_t bl = pack2(ctx_bl[s][2 * cp], ctx_bl[s][2 * cp + 1]);
        // r <= thr as the sign of r - thr - 1 (thr clamped to [-1, 32767]: r is in [0, 32767])
        const int tc = min(max(thr, -1), 32767);
        const uint32_t nthr = pack2(-(tc + 1), -(tc + 1));
        uint32_t kacc = 0;  // known counts per lane
        const uint32_t* ip = in2 + x / 2 + (size_t)ya * W2;
        uint32_t* op = out2 + x / 2 + (size_t)ya * W2;
        const size_t OS = SMEM ? (size_t)P5C : W2;  // scratch row stride
        const uint32_t* sp = SMEM ? scr + cp + (size_t)ya * P5C : op;
        auto row = [&](uint32_t v, uint32_t bw, uint32_t* dst) {
            const uint32_t mbw = sgn2(bw);
            const uint32_t b = (bl & mbw) | (bw & ~mbw);
            const uint32_t ma = sgn2(a), mab = ma | sgn2(b);
            const uint32_t mx = vmax2(a, b), mn = vmin2(a, b);
            const uint32_t r = vadd2(mx, vadd2(~mn, 0x00010001u));  // |a - b| (lanes with a, b >= 0)
            const uint32_t le = sgn2(vadd2(r, nthr));                // r <= thr
            const uint32_t avg = vadd2(a & b, ((a ^ b) >> 1) & 0x7fff7fffu);  // (a + b) >> 1, no overflow
            const uint32_t est = (avg & le) | (mn & ~le);
            const uint32_t edge = (et & ma) | (eb & ~ma);
            const uint32_t two = (edge & mab) | (est & ~mab);
            const uint32_t one = (b & ma) | (a & ~ma);
            const uint32_t u = (one & sg) | (two & ~sg);
            const uint32_t md = sgn2(v);
            const uint32_t res = (u & md) | (v & ~md);
            a = (a & md) | (v & ~md);
            *dst = res;
            kacc += (~res >> 15) & 0x00010001u;
        };
        // batches: all loads of P4B rows (input and scratch) issue before the
        // stores (the scratch loads would otherwise wait behind them)
        int y = ya;
        for (; y + P4B <= yb; y += P4B, ip += P4B * W2, op += P4B * W2, sp += P4B * OS) {
            uint32_t v[P4B], bw[P4B];
#pragma unroll
            for (int k = 0; k < P4B; ++k) {
                v[k] = __ldg(ip + k * W2);
                bw[k] = sp[k * OS];
            }
#pragma unroll
            for (int k = 0; k < P4B; ++k) row(v[k], bw[k], op + k * W2);
        }
        for (; y < yb; ++y, ip += W2, op += W2, sp += OS) row(__ldg(ip), *sp, op);
        known = (kacc & 0xffffu) + (kacc >> 16);
    }
    for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = known;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < P5C * P5S / 32; ++i) t += red[i];
        if (t) atomicAdd(&f.sc->known, t);
    }
}

// K6 v2: two rows per CTA in int16x2 lanes (row y in the low, row y+1 in
// the high half of every word): k_fill_rows16v's chunk / warp / block scans
// and its per-pixel rule, with lane masks by sign replication and LOP3
// selects -- one instruction per pixel pair where v1 spends one per pixel.
__global__ void __launch_bounds__(1024) k_fill_rows16p(Frame f, const int16_t* __restrict__ in,
                                                       int16_t* __restrict__ out,
                                                       const uint32_t* __restrict__ mbits) {
    __shared__ uint32_t wl[32], wf[32];
    const unsigned full = 0xffffffffu;
    const int W = f.W, y0 = 2 * blockIdx.x, tid = threadIdx.x;
    const bool two = y0 + 1 < f.H;
    const bool act = tid < W / 16;
    const int x0 = tid * 16;
    uint32_t P[16];
    {
        uint4 a0 = make_uint4(full, full, full, full), a1 = a0, b0 = a0, b1 = a0;
        if (act) {
            const uint4* s0 = reinterpret_cast<const uint4*>(in + (size_t)y0 * W + x0);
            a0 = __ldcs(s0);
            a1 = __ldcs(s0 + 1);
            if (two) {
                const uint4* s1 = reinterpret_cast<const uint4*>(in + (size_t)(y0 + 1) * W + x0);
                b0 = __ldcs(s1);
                b1 = __ldcs(s1 + 1);
            }
        }
        const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            P[2 * i] = __byte_perm(a[i], b[i], 0x5410);      // (row y px 2i, row y+1 px 2i)
            P[2 * i + 1] = __byte_perm(a[i], b[i], 0x7632);  // (.. px 2i+1 ..)
        }
        // frame path: the SAD writes only the matchable pixels (mbits) and
        // sparse is not pre-set, so every other pixel reads as unknown (-1)
        if (mbits) {
            uint32_t ma = 0, mb = 0;
            if (act) {
                ma = (__ldg(mbits + (size_t)y0 * f.bits_words + (x0 >> 5)) >> (x0 & 31)) & 0xffffu;
                if (two) mb = (__ldg(mbits + (size_t)(y0 + 1) * f.bits_words + (x0 >> 5)) >> (x0 & 31)) & 0xffffu;
            }
            const uint32_t keep = ma | (mb << 16);  // bit j: row y px j; bit 16 + j: row y+1 px j
#pragma unroll
            for (int j = 0; j < 16; ++j) P[j] |= ~((((keep >> j) & 0x10001u)) * 0xffffu);
        }
    }
    auto pick = [](uint32_t cur, uint32_t cand) {  // per lane: cur if known, else cand
        const uint32_t m = sgn2(cur);
        return (cand & m) | (cur & ~m);
    };
    uint32_t lastv = full, firstv = full;
#pragma unroll
    for (int i = 0; i < 16; ++i) lastv = pick(P[i], lastv);
#pragma unroll
    for (int i = 15; i >= 0; --i) firstv = pick(P[i], firstv);
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    uint32_t inc = lastv;  // latest known over lanes <= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(full, inc, o);
        if (lane >= o) inc = pick(inc, t);
    }
    uint32_t sinc = firstv;  // earliest known over lanes >= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_down_sync(full, sinc, o);
        if (lane + o < 32) sinc = pick(sinc, t);
    }
    if (lane == 31) wl[wid] = inc;
    if (lane == 0) wf[wid] = sinc;
    __syncthreads();
    uint32_t pd = __shfl_up_sync(full, inc, 1);
    if (lane == 0) pd = full;
    for (int i = wid - 1; i >= 0 && sgn2(pd); --i) pd = pick(pd, wl[i]);
    uint32_t nd = __shfl_down_sync(full, sinc, 1);
    if (lane == 31) nd = full;
    for (int i = wid + 1; i < nw && sgn2(nd); ++i) nd = pick(nd, wf[i]);
    if (!act) return;
    // right context of each pixel: the nearest known at or right of it
    uint32_t r[16];
#pragma unroll
    for (int i = 15; i >= 0; --i) {
        r[i] = nd;
        nd = pick(P[i], nd);
    }
    uint32_t o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        // unknown: filled iff nearest left == nearest right (both -1 -> stays -1)
        const uint32_t x = pd ^ r[i];
        const uint32_t eq = sgn2(__vadd2(x, full) & ~x);  // lanes with pd == r
        const uint32_t fillv = (pd & eq) | ~eq;           // pd where equal, else -1
        const uint32_t md = sgn2(P[i]);
        o[i] = (fillv & md) | (P[i] & ~md);
        pd = pick(P[i], pd);
    }
    uint4* d0 = reinterpret_cast<uint4*>(out + (size_t)y0 * W + x0);
    d0[0] = make_uint4(__byte_perm(o[0], o[1], 0x5410), __byte_perm(o[2], o[3], 0x5410),
                       __byte_perm(o[4], o[5], 0x5410), __byte_perm(o[6], o[7], 0x5410));
    d0[1] = make_uint4(__byte_perm(o[8], o[9], 0x5410), __byte_perm(o[10], o[11], 0x5410),
                       __byte_perm(o[12], o[13], 0x5410), __byte_perm(o[14], o[15], 0x5410));
    if (two) {
        uint4* d1 = reinterpret_cast<uint4*>(out + (size_t)(y0 + 1) * W + x0);
        d1[0] = make_uint4(__byte_perm(o[0], o[1], 0x7632), __byte_perm(o[2], o[3], 0x7632),
                           __byte_perm(o[4], o[5], 0x7632), __byte_perm(o[6], o[7], 0x7632));
        d1[1] = make_uint4(__byte_perm(o[8], o[9], 0x7632), __byte_perm(o[10], o[11], 0x7632),
                           __byte_perm(o[12], o[13], 0x7632), __byte_perm(o[14], o[15], 0x7632));
    }
}

}  // namespace

bool fill_rows_masks(int W) { return W % 16 == 0 && W <= 16384; }

void launch_fill_rows(const Frame& f, const int16_t* in, int16_t* out, cudaStream_t st, const uint32_t* mbits) {
    if (f.N == 0) return;
    if (fill_rows_masks(f.W)) {
        const int nt = ((f.W / 16) + 31) / 32 * 32;
        k_fill_rows16p<<<(f.H + 1) / 2, nt, 0, st>>>(f, in, out, mbits);
        return;
    }
    const size_t sm = (size_t)f.W * sizeof(int16_t);
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(k_fill_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_fill_rows<<<f.H, kFillThreads, sm, st>>>(f, in, out);
}

void launch_peek_cols(const Frame& f, const int16_t* in, int16_t* out, int16_t*, cudaStream_t st) {
    if (f.N == 0) return;
    if (f.W % 2 == 0 && (reinterpret_cast<uintptr_t>(in) & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
        // the scratch in shared memory when the strip fits (4K: 74 KB, 2 CTAs/SM)
        const size_t sm = (size_t)f.H * P5C * sizeof(uint32_t);
        if (sm <= 96 * 1024) {
            cudaFuncSetAttribute(k_peek_cols6<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_peek_cols6<true><<<(f.W + 2 * P5C - 1) / (2 * P5C), P5C * P5S, sm, st>>>(f, in, out);
        } else {
            k_peek_cols6<false><<<(f.W + 2 * P5C - 1) / (2 * P5C), P5C * P5S, 0, st>>>(f, in, out);
        }
        return;
    }
    k_peek_cols2<<<(f.W + PC - 1) / PC, PC * PS, 0, st>>>(f, in, out);
}

size_t peek_scratch_bytes(int, int) { return 0; }

}  // namespace stk
