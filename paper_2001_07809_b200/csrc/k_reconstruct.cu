// K6 fill_rows + K7 peek_cols -- dense reconstruction from the sparse map
// (reference: reconstruct.cpp:11-109, the paper's Algorithms 1 and 2).
//
// K6: one CTA per row; every thread owns a contiguous chunk (16 pixels in
//     registers when W % 16 == 0, else a shared-memory row), and two block
//     scans give each chunk the nearest known (x, d) on either side.  A run of
//     unknowns between consecutive knowns of equal disparity is filled; knowns
//     never change (reconstruct.cpp:11-33).
// K7: one CTA per 16 columns x 64 row segments (a warp = 16 columns x 2
//     segments: 32-byte row accesses).  Phase 1 summarises each
//     segment (known count, first/last known); phase 2 derives, per segment,
//     the nearest known above/below and, per column, the first two / last two
//     knowns; phase 3 walks the segment again and resolves each run of
//     unknowns with peek_estimate (reconstruct.cpp:40-46) on the snapshot:
//       0 knowns -> stays unknown, 1 known -> copy,
//       above & below -> est(above, below),
//       nothing above -> est(first two), nothing below -> est(last two).
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

// K6 v2: one CTA per row, thread = 16 consecutive pixels held in registers
// (2 x 16-byte loads / stores; W % 16 == 0, W <= 16384).  Block scans give
// every chunk the nearest known to its left (max-scan of (x+1) << 16 | d) and
// right (min-scan of x << 16 | d); the chunk is then filled in registers.
__global__ void __launch_bounds__(1024) k_fill_rows16(Frame f, const int16_t* __restrict__ in,
                                                      int16_t* __restrict__ out) {
    __shared__ uint32_t wl[32], wf[32];
    const int W = f.W, y = blockIdx.x, tid = threadIdx.x;
    const int nchunk = W / 16;
    const bool act = tid < nchunk;
    const int x0 = tid * 16;
    int16_t v[16];
    {
        uint4 a = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu), b = a;
        if (act) {
            const uint4* src = reinterpret_cast<const uint4*>(in + (size_t)y * W + x0);
            a = __ldcs(src);
            b = __ldcs(src + 1);
        }
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = (int16_t)(w[i >> 1] >> (16 * (i & 1)));
    }
    uint32_t klast = 0, kfirst = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (v[i] >= 0) klast = ((uint32_t)(x0 + i + 1) << 16) | (uint16_t)v[i];
#pragma unroll
    for (int i = 15; i >= 0; --i)
        if (v[i] >= 0) kfirst = ((uint32_t)(x0 + i) << 16) | (uint16_t)v[i];
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    uint32_t incl_l = klast;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl_l, o);
        if (lane >= o) incl_l = max(incl_l, t);
    }
    uint32_t incl_f = kfirst;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_down_sync(0xffffffffu, incl_f, o);
        if (lane + o < 32) incl_f = min(incl_f, t);
    }
    if (lane == 31) wl[wid] = incl_l;
    if (lane == 0) wf[wid] = incl_f;
    __syncthreads();
    uint32_t prev = __shfl_up_sync(0xffffffffu, incl_l, 1);
    if (lane == 0) prev = 0;
    for (int i = 0; i < wid; ++i) prev = max(prev, wl[i]);
    uint32_t next = __shfl_down_sync(0xffffffffu, incl_f, 1);
    if (lane == 31) next = 0xffffffffu;
    for (int i = wid + 1; i < nw; ++i) next = min(next, wf[i]);
    if (!act) return;
    // fill: a run of unknowns between knowns of equal disparity (the input
    // snapshot, reconstruct.cpp:11-33).  Left context: pd; right: the next known
    // inside the chunk or `next`.
    int pd = prev ? (int)(prev & 0xffffu) : -1;
    int nd[16];  // disparity of the nearest known at or right of i
    {
        int cur = next != 0xffffffffu ? (int)(next & 0xffffu) : -2;
#pragma unroll
        for (int i = 15; i >= 0; --i) {
            if (v[i] >= 0) cur = v[i];
            nd[i] = cur;
        }
    }
    int16_t o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (v[i] >= 0) {
            o[i] = v[i];
            pd = v[i];
        } else {
            o[i] = (pd >= 0 && nd[i] == pd) ? (int16_t)pd : (int16_t)-1;
        }
    }
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (uint16_t)o[2 * i] | ((uint32_t)(uint16_t)o[2 * i + 1] << 16);
    uint4* dst = reinterpret_cast<uint4*>(out + (size_t)y * W + x0);
    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
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

__global__ void __launch_bounds__(PC * PS) k_peek_cols(Frame f, const int16_t* __restrict__ in,
                                                       int16_t* __restrict__ out) {
    __shared__ SegSum seg[PS][PC];
    __shared__ unsigned long long red[PS];
    const int W = f.W, H = f.H, thr = f.thr;
    const int cx = threadIdx.x % PC, s = threadIdx.x / PC;
    const int x = blockIdx.x * PC + cx;
    const int sr = (H + PS - 1) / PS;
    const int ya = min(H, s * sr), yb = min(H, ya + sr);
    const bool col = x < W;
    // phase 1
    SegSum m{0, -1, -1, -1, -1};
    if (col)
        for (int yy = ya; yy < yb; yy += PB) {
            int16_t v[PB];
#pragma unroll
            for (int k = 0; k < PB; ++k) v[k] = yy + k < yb ? __ldg(in + (size_t)(yy + k) * W + x) : -1;
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                const int16_t d = v[k];
                if (d >= 0) {
                    if (m.count == 0) m.f1 = d;
                    else if (m.count == 1) m.f2 = d;
                    m.l2 = m.l1;
                    m.l1 = d;
                    ++m.count;
                }
            }
        }
    seg[s][cx] = m;
    __syncthreads();
    // phase 2
    int total = 0;
    for (int i = 0; i < PS; ++i) total += seg[i][cx].count;
    int above = -1, below = -1;
    for (int i = s - 1; i >= 0 && above < 0; --i)
        if (seg[i][cx].count) above = seg[i][cx].l1;
    for (int i = s + 1; i < PS && below < 0; ++i)
        if (seg[i][cx].count) below = seg[i][cx].f1;
    int cf1 = -1, cf2 = -1, cl1 = -1, cl2 = -1;  // column first two / last two
    for (int i = 0; i < PS && cf2 < 0; ++i) {
        const SegSum& g = seg[i][cx];
        if (!g.count) continue;
        if (cf1 < 0) {
            cf1 = g.f1;
            if (g.count > 1) cf2 = g.f2;
        } else {
            cf2 = g.f1;
        }
    }
    for (int i = PS - 1; i >= 0 && cl2 < 0; --i) {
        const SegSum& g = seg[i][cx];
        if (!g.count) continue;
        if (cl1 < 0) {
            cl1 = g.l1;
            if (g.count > 1) cl2 = g.l2;
        } else {
            cl2 = g.l1;
        }
    }
    // phase 3
    unsigned long long known = 0;
    if (col) {
        int cur = above;  // nearest known above the current run
        int rs = -1;      // first row of the pending run of unknowns
        auto resolve = [&](int nb, int y_end) {  // nb: nearest known below the run
            int16_t v;
            if (total == 0) v = -1;
            else if (total == 1) v = (int16_t)(cur >= 0 ? cur : nb);
            else if (cur >= 0 && nb >= 0) v = peek_estimate(cur, nb, thr);
            else if (cur < 0) v = peek_estimate(cf1, cf2, thr);
            else v = peek_estimate(cl2, cl1, thr);
            for (int q = rs; q < y_end; ++q) out[(size_t)q * W + x] = v;
            if (v >= 0) known += (unsigned long long)(y_end - rs);
            rs = -1;
        };
        for (int yy = ya; yy < yb; yy += PB) {
            int16_t v[PB];
#pragma unroll
            for (int k = 0; k < PB; ++k) v[k] = yy + k < yb ? __ldg(in + (size_t)(yy + k) * W + x) : -1;
#pragma unroll
            for (int k = 0; k < PB; ++k) {
                const int y = yy + k;
                if (y >= yb) break;
                const int16_t d = v[k];
                if (d < 0) {
                    if (rs < 0) rs = y;
                    continue;
                }
                if (rs >= 0) resolve(d, y);
                out[(size_t)y * W + x] = d;
                ++known;
                cur = d;
            }
        }
        if (rs >= 0) resolve(below, yb);
    }
    // known count for DepthStats::known_fraction
    for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = known;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < PC * PS / 32; ++i) t += red[i];
        if (t) atomicAdd(&f.sc->known, t);
    }
}

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

// K7 v4: k_peek_cols2's algorithm with two adjacent columns per thread
// (32-bit loads/stores of int16 pairs: a warp's 8 column pairs x 4 segments
// move 32 contiguous bytes per row each) and unchecked full batches.
constexpr int P4C = 8;   // column pairs per CTA (16 columns)
constexpr int P4S = 64;  // row segments per column
constexpr int P4B = 8;   // rows per batch

struct ColSeg {  // segment summary of one column while walking down
    int count, f1, f2, l1, l2;
};
__device__ __forceinline__ void seg_add(ColSeg& m, int d) {
    const bool kn = d >= 0;
    m.f2 = (kn && m.count == 1) ? d : m.f2;
    m.f1 = (kn && m.count == 0) ? d : m.f1;
    m.l2 = kn ? m.l1 : m.l2;
    m.l1 = kn ? d : m.l1;
    m.count += kn;
}
__device__ __forceinline__ uint32_t pack2(int a, int b) { return (uint32_t)(uint16_t)a | (uint32_t)b << 16; }
__device__ __forceinline__ int lo16(uint32_t v) { return (int16_t)(v & 0xffffu); }
__device__ __forceinline__ int hi16s(uint32_t v) { return (int16_t)(v >> 16); }

__global__ void __launch_bounds__(P4C * P4S, 2) k_peek_cols4(Frame f, const int16_t* __restrict__ in,
                                                          int16_t* __restrict__ out) {
    __shared__ SegSum seg[P4S][2 * P4C];
    __shared__ int16_t ctx_ab[P4S][2 * P4C], ctx_bl[P4S][2 * P4C];
    __shared__ int col_total[2 * P4C], col_top[2 * P4C], col_bot[2 * P4C];
    __shared__ unsigned long long red[P4C * P4S / 32];
    const int W = f.W, H = f.H, thr = f.thr;
    const int cp = threadIdx.x % P4C, s = threadIdx.x / P4C;
    const int x = 2 * (blockIdx.x * P4C + cp);  // W even
    const int sr = (H + P4S - 1) / P4S;
    const int ya = min(H, s * sr), yb = min(H, ya + sr);
    const bool col = x < W;
    const uint32_t* __restrict__ in2 = reinterpret_cast<const uint32_t*>(in);
    uint32_t* __restrict__ out2 = reinterpret_cast<uint32_t*>(out);
    const size_t W2 = (size_t)W / 2;  // row stride in pairs
    // pass 1 (top-down)
    ColSeg m0{0, -1, -1, -1, -1}, m1{0, -1, -1, -1, -1};
    if (col) {
        int c0 = -1, c1 = -1;
        size_t o = (size_t)ya * W2 + x / 2;
        for (int yy = ya; yy < yb; yy += P4B, o += P4B * W2) {
            const int n = min(P4B, yb - yy);
            uint32_t v[P4B];
            if (n == P4B) {
#pragma unroll
                for (int k = 0; k < P4B; ++k) v[k] = __ldg(in2 + o + k * W2);
#pragma unroll
                for (int k = 0; k < P4B; ++k) {
                    out2[o + k * W2] = pack2(c0, c1);
                    const int d0 = lo16(v[k]), d1 = hi16s(v[k]);
                    seg_add(m0, d0);
                    seg_add(m1, d1);
                    c0 = d0 >= 0 ? d0 : c0;
                    c1 = d1 >= 0 ? d1 : c1;
                }
            } else {
                for (int k = 0; k < n; ++k) {
                    const uint32_t vk = __ldg(in2 + o + k * W2);
                    out2[o + k * W2] = pack2(c0, c1);
                    const int d0 = lo16(vk), d1 = hi16s(vk);
                    seg_add(m0, d0);
                    seg_add(m1, d1);
                    c0 = d0 >= 0 ? d0 : c0;
                    c1 = d1 >= 0 ? d1 : c1;
                }
            }
        }
    }
    seg[s][2 * cp] = SegSum{m0.count, (int16_t)m0.f1, (int16_t)m0.f2, (int16_t)m0.l1, (int16_t)m0.l2};
    seg[s][2 * cp + 1] = SegSum{m1.count, (int16_t)m1.f1, (int16_t)m1.f2, (int16_t)m1.l1, (int16_t)m1.l2};
    __syncthreads();
    // phase 2: one thread per column scans the segments once
    if (threadIdx.x < 2 * P4C) {
        const int cx = threadIdx.x;
        int total = 0, last = -1, cf1 = -1, cf2 = -1;
        for (int i = 0; i < P4S; ++i) {
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
        for (int i = P4S - 1; i >= 0; --i) {
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
    // pass 2 (bottom-up)
    unsigned long long known = 0;
    if (col) {
        const int t0 = col_total[2 * cp], t1 = col_total[2 * cp + 1];
        const int et0 = col_top[2 * cp], et1 = col_top[2 * cp + 1];
        const int eb0 = col_bot[2 * cp], eb1 = col_bot[2 * cp + 1];
        const int ab0 = ctx_ab[s][2 * cp], ab1 = ctx_ab[s][2 * cp + 1];
        int nb0 = ctx_bl[s][2 * cp], nb1 = ctx_bl[s][2 * cp + 1];
        auto resolve = [&](int d, int a, int above, int& nb, int total, int et, int eb) {
            const int ab = a >= 0 ? a : above;  // nearest known above
            int r;
            if (d >= 0) r = d;
            else if (total == 0) r = -1;
            else if (total == 1) r = ab >= 0 ? ab : nb;
            else if (ab >= 0 && nb >= 0) r = peek_estimate(ab, nb, thr);
            else r = ab < 0 ? et : eb;
            nb = d >= 0 ? d : nb;
            return r;
        };
        for (int yy = yb - 1; yy >= ya; yy -= P4B) {
            const int n = min(P4B, yy - ya + 1);
            const size_t o = (size_t)yy * W2 + x / 2;
            if (n == P4B) {
                uint32_t v[P4B], a[P4B];
#pragma unroll
                for (int k = 0; k < P4B; ++k) {
                    v[k] = __ldg(in2 + o - k * W2);
                    a[k] = out2[o - k * W2];
                }
#pragma unroll
                for (int k = 0; k < P4B; ++k) {
                    const int r0 = resolve(lo16(v[k]), lo16(a[k]), ab0, nb0, t0, et0, eb0);
                    const int r1 = resolve(hi16s(v[k]), hi16s(a[k]), ab1, nb1, t1, et1, eb1);
                    out2[o - k * W2] = pack2(r0, r1);
                    known += (r0 >= 0) + (r1 >= 0);
                }
            } else {
                for (int k = 0; k < n; ++k) {
                    const uint32_t vk = __ldg(in2 + o - k * W2), ak = out2[o - k * W2];
                    const int r0 = resolve(lo16(vk), lo16(ak), ab0, nb0, t0, et0, eb0);
                    const int r1 = resolve(hi16s(vk), hi16s(ak), ab1, nb1, t1, et1, eb1);
                    out2[o - k * W2] = pack2(r0, r1);
                    known += (r0 >= 0) + (r1 >= 0);
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = known;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < P4C * P4S / 32; ++i) t += red[i];
        if (t) atomicAdd(&f.sc->known, t);
    }
}

}  // namespace

void launch_fill_rows(const Frame& f, const int16_t* in, int16_t* out, cudaStream_t st) {
    if (f.N == 0) return;
    if (f.W % 16 == 0 && f.W <= 16384) {
        const int nt = ((f.W / 16) + 31) / 32 * 32;
        k_fill_rows16<<<f.H, nt, 0, st>>>(f, in, out);
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
        k_peek_cols4<<<(f.W + 2 * P4C - 1) / (2 * P4C), P4C * P4S, 0, st>>>(f, in, out);
        return;
    }
    k_peek_cols2<<<(f.W + PC - 1) / PC, PC * PS, 0, st>>>(f, in, out);
}

size_t peek_scratch_bytes(int, int) { return 0; }

}  // namespace stk
