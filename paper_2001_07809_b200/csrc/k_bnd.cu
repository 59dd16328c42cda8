// K3b/K4b -- bit-packed boundary stage of the frame path (reference:
// boundary.cpp:11-195, pipeline.cpp:87-94).  Every mask is a 32-bit word per
// 32 pixels of a row (bit x & 31 of word x >> 5), so the morphology is a few
// word-wide logic ops per 32 pixels and the connected components work on runs
// instead of pixels: no per-pixel label / parent array is ever written.
//
//   B1 morph_bits   gray -> K-Means label bit-planes (on chip, via the LUT) ->
//                   detect (any Moore neighbour label differs) -> fill ->
//                   remove, one warp per 30 word-columns x 32 rows, rows
//                   streamed with a 3-row halo; refined bits + raw/refined
//                   counts (raw bytes too in full mode).
//   B2 ccl_region   CTA per 256x128 region, warp per 32x32 tile: run-level
//                   union-find per tile, then the region's inner tile borders
//                   merged in shared memory; every region component goes to
//                   the root list with its size and its minimum raster index g
//                   (par[g] = g, the global union-find node); each run records
//                   its component's g, the region's outer borders the g of
//                   their pixels.
//   B3 ccl_borders  CTA per region: top-border pixels unite with their three
//                   neighbours in the regions above, left-border pixels with
//                   the left region (lock-free union, hash-priority linking,
//                   path halving).
//   B4-B7 prune_fused  one cooperative launch, grid barriers between:
//                   compress region roots (dense ids) to global roots with
//                   size and minimum raster index (the reference's discovery
//                   order) summed / min'ed at the root; size histogram;
//                   s* = smallest size whose class-cumulative pixel count
//                   exceeds B = floor(budget), q = floor((B - CS(s*-1)) / s*);
//                   size < s* removed; size == s* -> bit (min raster index) of
//                   a bitmap whose first q set bits in raster (= label) order
//                   are removed by one ordered scan.
//   B8 apply_runs   warp per tile: runs -> their root -> removed?  -> pruned
//                   bits, border anchors, window filter -> matchable bits and
//                   the frame counts (bytes in full mode).
//   B9 list_bits    (only for the per-pixel SAD list kernel) ordered
//                   compaction of the matchable bits.
#include <cub/device/device_scan.cuh>
#include <cstdlib>

#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int CT = 32;         // CCL tile side
constexpr int kRunCap = 512;   // max runs in a 32x32 tile (16 per row): runroot stride
constexpr int kRunCapFast = 224;  // B2's shared-memory run table (overflow tiles: second pass)
#ifndef STK_MB_ROWS
#define STK_MB_ROWS 8
#endif
// B1 output rows per warp (STK_MB_ROWS: experiment knob; 4K: 4 rows 18.1 us, 6: 17.9, 8: 17.1, 12: 18.8)
constexpr int MB_ROWS = STK_MB_ROWS;
constexpr int MB_WPW = 30;     // B1 output words per warp (+1 halo word each side)

__device__ __forceinline__ uint32_t upto_mask(int j) {  // bits 0..j
    return j >= 31 ? 0xffffffffu : ((2u << j) - 1u);
}

__device__ __forceinline__ int run_len(uint32_t m, int a) {  // set bits from a upward
    const uint32_t inv = ~(m >> a);
    return inv ? __ffs(inv) - 1 : 32 - a;
}

__device__ __forceinline__ uint32_t bits_to_bytes4(uint32_t nib) {  // 4 bits -> 4 bytes 0/1
    return (nib * 0x00204081u) & 0x01010101u;
}

__device__ __forceinline__ void store_bits_as_bytes(uint8_t* dst, uint32_t v) {  // 32 bytes
    uint4 a, b;
    a.x = bits_to_bytes4(v & 15u), a.y = bits_to_bytes4((v >> 4) & 15u);
    a.z = bits_to_bytes4((v >> 8) & 15u), a.w = bits_to_bytes4((v >> 12) & 15u);
    b.x = bits_to_bytes4((v >> 16) & 15u), b.y = bits_to_bytes4((v >> 20) & 15u);
    b.z = bits_to_bytes4((v >> 24) & 15u), b.w = bits_to_bytes4(v >> 28);
    reinterpret_cast<uint4*>(dst)[0] = a;
    reinterpret_cast<uint4*>(dst)[1] = b;
}

__device__ __forceinline__ int gfind(int* p, int x) {  // path halving
    int q = __ldcg(p + x);
    while (q != x) {
        const int g = __ldcg(p + q);
        if (g != q) p[x] = g;
        x = q;
        q = g;
    }
    return x;
}

// Read-only find for the compress passes after the union phase: a thread
// then writes only final roots (par[id] = root), so no concurrent path-
// halving store can overwrite an already-compressed entry with an
// intermediate node (a race gfind would have there).
__device__ __forceinline__ int gfind_ro(const int* p, int x) {
    int q = __ldcg(p + x);
    while (q != x) {
        x = q;
        q = __ldcg(p + x);
    }
    return x;
}

// Programmatic dependent launch: the boundary chain's kernels (B2 ... B8)
// start with a grid-dependency wait (a no-op without the launch attribute)
// and are launched with programmatic stream serialisation, so each one's
// CTAs are scheduled while its predecessor still runs and only the wait
// separates them: boundary stage 0.115 -> 0.103 ms, frames/s unchanged
// (STK_PDL=0: plain launches, the A/B switch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Global union-find over region roots: link by a hash priority of the node
// (random-permutation order keeps the trees O(log n) deep even for one giant
// component); the component's minimum raster index is tracked separately
// (minkey) because the reference's label order needs it, not the root.
__device__ __forceinline__ uint32_t prio(int x) {
    uint32_t h = (uint32_t)x * 0x9E3779B1u;  // odd multiplier and xor-shift: bijective
    h ^= h >> 15;
    h *= 0x85EBCA77u;
    h ^= h >> 13;
    return h;
}

__device__ __forceinline__ void gunite(int* p, int a, int b) {
    while (true) {
        a = gfind(p, a);
        b = gfind(p, b);
        if (a == b) return;
        if (prio(a) < prio(b)) {
            const int t = a;
            a = b;
            b = t;
        }
        // link b (lower priority) under a, if b is still a root
        if (atomicCAS(p + b, b, a) == b) return;
    }
}

// a united with up to 3 nodes b[0..nb): the 1 + nb root walks (path halving)
// advance in lockstep, so their dependent L2 loads overlap instead of running
// one chain after another; then the roots are linked by priority (CAS), a
// lost race falls back to gunite.
__device__ __forceinline__ void gunite_n(int* p, int a, const int (&b)[3], int nb) {
    int x[4] = {a, b[0], b[1], b[2]};
    bool act[4] = {true, nb > 0, nb > 1, nb > 2};
    while (act[0] | act[1] | act[2] | act[3]) {
        int q[4], g[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (act[i]) q[i] = __ldcg(p + x[i]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!act[i]) continue;
            if (q[i] == x[i]) act[i] = false;
            else g[i] = __ldcg(p + q[i]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!act[i]) continue;
            if (g[i] == q[i]) {
                x[i] = q[i];
                act[i] = false;
            } else {
                p[x[i]] = g[i];
                x[i] = g[i];
            }
        }
    }
    int r = x[0];
#pragma unroll
    for (int i = 1; i < 4; ++i) {
        if (i > nb) break;
        const int rb = x[i];
        if (rb == r || (i > 1 && rb == x[1]) || (i > 2 && rb == x[2])) continue;
        const int hi = prio(r) > prio(rb) ? r : rb, lo = r ^ rb ^ hi;
        if (atomicCAS(p + lo, lo, hi) == lo) {
            r = hi;
        } else {
            gunite(p, r, rb);
            r = gfind(p, r);
        }
    }
}

// ------------------------------------------------------------------ B1 ----
// NPL label bit-planes.  lutp[v] holds bit p of lut[v] at bit 8p (p < 4), so
// 8 pixels combine with shift-adds into one word whose byte p is plane p's
// 8 bits; planes 4..7 use lutq the same way.
//
// MODE selects where the streamed rows enter the detect -> fill -> remove
// pipeline (same word ops, same edge rules, same row schedule):
//   MB_FRAME   gray (pitched u8) -> K-Means LUT planes -> detect -> fill ->
//              remove -> refined bits (+ raw bytes in full mode); the frame path
//   MB_DET16   u16 labels (pitch 2P) -> planes poff..poff+NPL-1 -> detect ->
//              raw bits (OR-ed in when poff > 0); detect_boundaries entry
//   MB_FILL    byte mask -> (as raw bits) fill -> filled bits; morph_fill entry
//   MB_REMOVE  byte mask -> (as filled bits) remove -> bits; morph_remove entry
enum { MB_FRAME = 0, MB_DET16 = 1, MB_FILL = 2, MB_REMOVE = 3 };

__device__ __forceinline__ uint32_t bytes_nz_bits(const uint4 (&g)[2]) {  // 32 bytes -> 32 bits (!= 0)
    const uint32_t w8[8] = {g[0].x, g[0].y, g[0].z, g[0].w, g[1].x, g[1].y, g[1].z, g[1].w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t t = __vcmpne4(w8[i], 0u) & 0x01010101u;  // flag of byte b at bit 8b
        m |= ((t | (t >> 7) | (t >> 14) | (t >> 21)) & 0xfu) << (4 * i);
    }
    return m;
}

template <int NPL, int MODE>
__global__ void __launch_bounds__(128) k_morph_bits(Frame f, uint32_t* __restrict__ rbits,
                                                    const uint8_t* __restrict__ src, int poff) {
    constexpr int NQ = MODE == MB_DET16 ? 4 : 2;  // uint4 per 32-pixel word column
    __shared__ uint32_t lutp[256], lutq[256];
    __shared__ unsigned long long red[2][4];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if constexpr (MODE == MB_FRAME) {
        for (int v = tid; v < 256; v += blockDim.x) {
            const uint32_t l = f.sc->lut[v];
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                a |= ((l >> p) & 1u) << (8 * p);
                b |= ((l >> (p + 4)) & 1u) << (8 * p);
            }
            lutp[v] = a;
            lutq[v] = b;
        }
        __syncthreads();
        src = f.grayL;
    }
    const size_t pitch = MODE == MB_DET16 ? 2 * (size_t)f.P : (size_t)f.P;
    const int W = f.W, H = f.H, BW = (W + 31) >> 5;
    const int strips = (BW + MB_WPW - 1) / MB_WPW;
    const int gw = blockIdx.x * 4 + wid;
    const int strip = gw % strips, band = gw / strips;
    const int yb = band * MB_ROWS;
    unsigned long long n_raw = 0, n_ref = 0;
    if (yb < H) {
        const int wc = strip * MB_WPW - 1 + lane;                // this lane's word column
        const bool out_lane = lane >= 1 && lane <= MB_WPW && wc < BW;
        const int wcl = min(max(wc, 0), BW - 1);                 // clamped for loads
        const bool first = wc == 0, last = wc == BW - 1;
        // bits of this word inside the image
        const int nvalid = W - 32 * wc;
        const uint32_t valid = nvalid >= 32 ? 0xffffffffu : (nvalid > 0 ? (1u << nvalid) - 1u : 0u);
        // interior columns 1..W-2
        uint32_t icol = valid;
        if (first) icol &= ~1u;
        if (nvalid >= 1 && nvalid <= 32) icol &= ~(1u << (nvalid - 1));
        const int replb = (W - 1) & 31;  // bit of pixel W-1 in the last word

        auto shl = [&](uint32_t v) {  // bit x <- pixel x-1 (replicate at x = 0)
            const uint32_t l = __shfl_up_sync(0xffffffffu, v, 1);
            return (v << 1) | (first ? (v & 1u) : (l >> 31));
        };
        auto shr = [&](uint32_t v) {  // bit x <- pixel x+1 (replicate at the right edge)
            const uint32_t r = __shfl_down_sync(0xffffffffu, v, 1);
            return (v >> 1) | ((last ? (v >> 31) : (r & 1u)) << 31);
        };
        // rows are fetched two iterations ahead of their use (load latency)
        auto load_row = [&](int ri, uint4 (&g)[NQ]) {
            ri = min(max(ri, 0), H - 1);
            const uint4* p = reinterpret_cast<const uint4*>(src + (size_t)ri * pitch + 16 * NQ * wcl);
#pragma unroll
            for (int q = 0; q < NQ; ++q) g[q] = __ldg(p + q);
        };
        auto planes_of = [&](const uint4 (&gq)[NQ], uint32_t (&pl)[NPL]) {
#pragma unroll
            for (int p = 0; p < NPL; ++p) pl[p] = 0;
            if constexpr (MODE == MB_FRAME) {
                const uint4 g0 = gq[0], g1 = gq[1];
                const uint32_t gw8[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
                for (int oct = 0; oct < 4; ++oct) {
                    uint32_t a = 0, b = 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t v = (gw8[2 * oct + (i >> 2)] >> (8 * (i & 3))) & 0xffu;
                        a += lutp[v] << i;
                        if (NPL > 4) b += lutq[v] << i;
                    }
#pragma unroll
                    for (int p = 0; p < NPL; ++p) {
                        const uint32_t byte = p < 4 ? (a >> (8 * p)) & 0xffu : (b >> (8 * (p - 4))) & 0xffu;
                        pl[p] |= byte << (8 * oct);
                    }
                }
            } else if constexpr (MODE == MB_DET16) {
                uint32_t w16[16];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    w16[4 * q] = gq[q].x, w16[4 * q + 1] = gq[q].y;
                    w16[4 * q + 2] = gq[q].z, w16[4 * q + 3] = gq[q].w;
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const uint32_t lab = ((w16[i >> 1] >> (16 * (i & 1))) & 0xffffu) >> poff;
#pragma unroll
                    for (int p = 0; p < NPL; ++p) pl[p] |= ((lab >> p) & 1u) << i;
                }
            }
            if (last && nvalid < 32) {  // pixels beyond W replicate pixel W-1
#pragma unroll
                for (int p = 0; p < NPL; ++p) pl[p] = (pl[p] & valid) | (((pl[p] >> replb) & 1u) ? ~valid : 0u);
            }
        };
        // sliding windows: label planes (3 rows + shifted), raw (3 rows), fill (3 rows)
        uint32_t P0[NPL], P1[NPL], P2[NPL], L1[NPL], R1[NPL], L0[NPL], R0[NPL], L2[NPL], R2[NPL];
        uint32_t raw0 = 0, raw1 = 0, raw2 = 0, fil0 = 0, fil1 = 0, fil2 = 0;
        uint32_t m0 = 0, m1 = 0, m2 = 0;  // mask modes: bits of rows ri, ri-1, ri-2
        uint4 qa[NQ], qb[NQ], qc[NQ];
        load_row(yb - 3, qa);
        load_row(yb - 2, qb);
        for (int i = 0; i < MB_ROWS + 6; ++i) {
            const int ri = yb - 3 + i;
            if constexpr (MODE == MB_FILL || MODE == MB_REMOVE) {
                m2 = m1;
                m1 = m0;
                m0 = bytes_nz_bits(qa) & valid;  // row ri (qa holds row ri)
                load_row(ri + 2, qc);
#pragma unroll
                for (int q = 0; q < NQ; ++q) qa[q] = qb[q], qb[q] = qc[q];
            } else {
                // shift the plane window: (P0, P1, P2) = rows ri-2, ri-1, ri
#pragma unroll
                for (int p = 0; p < NPL; ++p) {
                    P0[p] = P1[p], L0[p] = L1[p], R0[p] = R1[p];
                    P1[p] = P2[p], L1[p] = L2[p], R1[p] = R2[p];
                }
                load_row(ri + 2, qc);
                planes_of(qa, P2);
#pragma unroll
                for (int q = 0; q < NQ; ++q) qa[q] = qb[q], qb[q] = qc[q];
#pragma unroll
                for (int p = 0; p < NPL; ++p) {
                    L2[p] = shl(P2[p]);
                    R2[p] = shr(P2[p]);
                }
            }
            if (i < 2) continue;
            // detect row rd = ri - 1 (planes rows ri-2, ri-1, ri)
            const int rd = ri - 1;
            uint32_t rawn;
            if constexpr (MODE == MB_FILL || MODE == MB_REMOVE) {
                rawn = rd >= 0 && rd < H ? m1 : 0u;  // the input mask enters as the raw rows
            } else {
                uint32_t diff = 0;
#pragma unroll
                for (int p = 0; p < NPL; ++p) {
                    const uint32_t c = P1[p];
                    diff |= (c ^ P0[p]) | (c ^ L0[p]) | (c ^ R0[p]) | (c ^ L1[p]) | (c ^ R1[p]) |
                            (c ^ P2[p]) | (c ^ L2[p]) | (c ^ R2[p]);
                }
                rawn = rd >= 0 && rd < H ? diff & valid : 0u;
            }
            if (out_lane && rd >= yb && rd < yb + MB_ROWS && rd < H) {
                n_raw += __popc(rawn);
                if constexpr (MODE == MB_FRAME) {
                    if (f.full) store_bits_as_bytes(f.mraw + (size_t)rd * f.P + 32 * wc, rawn);
                } else if constexpr (MODE == MB_DET16) {
                    uint32_t* o = rbits + (size_t)rd * f.bits_words + wc;
                    *o = poff ? (*o | rawn) : rawn;
                }
            }
            if constexpr (MODE == MB_DET16) continue;
            raw0 = raw1, raw1 = raw2, raw2 = rawn;  // rows rd-2, rd-1, rd
            if (i < 4) continue;
            // fill row rf = rd - 1 (raw rows rd-2, rd-1, rd)
            const int rf = rd - 1;
            uint32_t filn = raw1;
            if constexpr (MODE == MB_REMOVE) {
                filn = rf >= 0 && rf < H ? m2 : 0u;  // the input mask enters as the filled rows
            } else if (rf >= 1 && rf <= H - 2) {
                const uint32_t all8 = raw0 & shl(raw0) & shr(raw0) & shl(raw1) & shr(raw1) & raw2 &
                                      shl(raw2) & shr(raw2);
                filn |= all8 & icol;
            }
            if constexpr (MODE == MB_FILL) {
                if (out_lane && rf >= yb && rf < yb + MB_ROWS && rf < H)
                    rbits[(size_t)rf * f.bits_words + wc] = filn;
                continue;
            }
            fil0 = fil1, fil1 = fil2, fil2 = filn;  // rows rf-2, rf-1, rf
            if (i < 6) continue;
            // remove row rr = rf - 1 (fill rows rf-2, rf-1, rf)
            const int rr = rf - 1;
            uint32_t refn = fil1;
            const uint32_t l4 = shl(fil1), r4 = shr(fil1);
            if (rr >= 1 && rr <= H - 2) refn &= ~(fil0 & fil2 & l4 & r4 & icol);
            if (out_lane && rr >= yb && rr < H) {
                rbits[(size_t)rr * f.bits_words + wc] = refn;
                n_ref += __popc(refn);
            }
        }
    }
    if constexpr (MODE != MB_FRAME) return;
    for (int o = 16; o > 0; o >>= 1) {
        n_raw += __shfl_xor_sync(0xffffffffu, n_raw, o);
        n_ref += __shfl_xor_sync(0xffffffffu, n_ref, o);
    }
    if (lane == 0) {
        red[0][wid] = n_raw;
        red[1][wid] = n_ref;
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned long long a = red[0][0] + red[0][1] + red[0][2] + red[0][3];
        const unsigned long long b = red[1][0] + red[1][1] + red[1][2] + red[1][3];
        if (a) atomicAdd(&f.sc->raw_count, a);
        if (b) atomicAdd(&f.sc->refined_count, b);
    }
}

// Stage entries: B1's result bits -> the reference's bytes.  detect: 0/1;
// fill: out = mask copy with filled zeros set to 1 (boundary.cpp:42, :58);
// remove: out = mask copy with removed pixels cleared (boundary.cpp:66, :81).
template <int MODE>
__global__ void __launch_bounds__(256) k_bits_to_bytes(Frame f, const uint32_t* __restrict__ rbits,
                                                       const uint8_t* __restrict__ in,
                                                       uint8_t* __restrict__ out) {
    const int BW = (f.W + 31) / 32;
    const long long nw = (long long)BW * f.H;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nw;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / BW), wc = (int)(i - (long long)y * BW);
        const uint32_t b = rbits[(size_t)y * f.bits_words + wc];
        uint8_t* o = out + (size_t)y * f.P + 32 * wc;
        if constexpr (MODE == MB_DET16) {
            store_bits_as_bytes(o, b);
        } else {
            const uint4* ip = reinterpret_cast<const uint4*>(in + (size_t)y * f.P + 32 * wc);
            uint4 v[2] = {ip[0], ip[1]};
            uint32_t* vw = reinterpret_cast<uint32_t*>(v);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t flag = bits_to_bytes4((b >> (4 * k)) & 15u);  // 0/1 bytes
                if constexpr (MODE == MB_FILL) vw[k] = vw[k] | (flag & ~__vcmpne4(vw[k], 0u));
                else vw[k] &= flag * 0xffu;
            }
            reinterpret_cast<uint4*>(o)[0] = v[0];
            reinterpret_cast<uint4*>(o)[1] = v[1];
        }
    }
}

__device__ __forceinline__ unsigned long long budget_of(const Frame& f) {
    // boundary.cpp:156: fraction * double(mask.count()); integer sizes compare
    // <= budget  <=>  <= floor(budget)
    return (unsigned long long)floor(__dmul_rn(f.frac, (double)f.sc->refined_count));
}

// ------------------------------------------------------------------ B2 ----
// One CTA per region of RGX x RGY tiles (one warp per 32x32 tile).
//  1. tile-local CCL: runs are numbered in (row, start) order (ridx); lanes
//     work on runs ridx = lane, lane + 32, ... so the union-find phases stay
//     converged; 8-connected unions with the overlapping runs of the row
//     above; min-linking makes a component's root its first run, i.e. its
//     minimum raster index.
//  2. region merge in shared memory: node = warp * CAP + ridx; the tiles'
//     inner borders are united, and every region component gets the minimum
//     raster index g of its tile components (its key) and their size sum.
//  3. region components -> root list (g, size), par[g] = g; every run records
//     its component's g; the region's outer borders record the g of their
//     pixels for the global merge (B3).
// region = RGX x RGY tiles (STK_RGX / STK_RGY: experiment knobs; 4 x 2: boundary
// stage 0.165 ms, 4 x 4: 0.150 ms -- half the borders left for B3; with B3b's
// edge list, 4 x 4: 0.134 ms, 4 x 8: 0.128, 8 x 4: 0.126 -- fewer edges to unite)
#ifndef STK_RGX
#define STK_RGX 8
#endif
#ifndef STK_RGY
#define STK_RGY 4
#endif
constexpr int RGX = STK_RGX, RGY = STK_RGY, NRW = RGX * RGY;  // 256 x 128-pixel regions
constexpr int RW = RGX * CT, RH = RGY * CT;
constexpr int RBORD = 2 * RW + 2 * RH;             // [top RW][bottom RW][left RH][right RH]

// Per-tile run table; the union-find arrays are region-wide and flat (node
// w * CAP + ridx indexes them directly: no struct-stride address math in the
// finds -- 14.9 % of B2's instructions went to R[node / CAP].par[node % CAP])
template <int CAP>
struct RunSmemT {
    uint32_t rowm[CT], rows[CT];   // row masks, run starts
    int rs[CT + 1];                // first ridx of each row
    uint8_t rstart[CAP], rlen[CAP], rrow[CAP];
};

// shared memory of a B2 CTA: [NRW tile tables][par][key][sz], the last three
// NRW * CAP entries each: par = region node ids after step 1, key = g of the
// tile-local roots (INT_MAX otherwise), sz = sizes (u16: a region's
// components hold <= 256 x 128 pixels)
template <int CAP>
constexpr size_t region_smem_bytes() {
    return NRW * (sizeof(RunSmemT<CAP>) + (size_t)CAP * (2 * sizeof(int) + sizeof(uint16_t)));
}

// sz[i] += v: a 32-bit shared atomic on the u16's word (v and the sums stay
// below 2^16, so the low half never carries into the high one; sz is 4-byte
// aligned)
__device__ __forceinline__ void sz_add(uint16_t* sz, int i, unsigned v) {
    atomicAdd(reinterpret_cast<unsigned*>(&sz[i & ~1]), v << (16 * (i & 1)));
}

__device__ __forceinline__ int rfind(int* p, int x) {  // with path halving
    int q = p[x];
    while (q != x) {
        const int g = p[q];
        if (g != q) p[x] = g;
        x = q;
        q = g;
    }
    return x;
}

__device__ __forceinline__ void runite(int* p, int a, int b) {
    while (true) {
        a = rfind(p, a);
        b = rfind(p, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(&p[b], a);
        if (old == b) return;
        b = old;
    }
}

// region node of pixel (row, col) of warp w's tile, -1 when unset
template <int CAP>
__device__ __forceinline__ int node_at(const RunSmemT<CAP>* R, int w, int row, int col) {
    const RunSmemT<CAP>& S = R[w];
    if (!((S.rowm[row] >> col) & 1u)) return -1;
    return w * CAP + S.rs[row] + __popc(S.rows[row] & upto_mask(col)) - 1;
}

// Region body: CAP = the run table's per-tile capacity.  FIRST (CAP = 224):
// a region with a tile of more runs appends itself to the overflow list
// (f.list, count in sc->n_ovf) and writes nothing; the overflow pass (CAP =
// 512, the most a 32x32 tile can hold) then runs those regions.
template <int CAP, bool FIRST>
__device__ __forceinline__ void ccl_region_body(const Frame& f, const uint32_t* __restrict__ rbits,
                                                int32_t* __restrict__ runroot, int32_t* __restrict__ bord,
                                                int reg, uint8_t* smraw) {
    using RunSmem = RunSmemT<CAP>;
    RunSmem* R = reinterpret_cast<RunSmem*>(smraw);
    int* P = reinterpret_cast<int*>(smraw + NRW * sizeof(RunSmem));  // region-wide, node-indexed
    int* KY = P + NRW * CAP;
    uint16_t* SZ = reinterpret_cast<uint16_t*>(KY + NRW * CAP);
    __shared__ int s_ovf;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TXc = (f.W + CT - 1) / CT, TYc = (f.H + CT - 1) / CT;
    const int RXc = (f.W + RW - 1) / RW;
    const int rx = reg % RXc, ry = reg / RXc;
    const int tc = wid % RGX, tr = wid / RGX;
    const int tx = rx * RGX + tc, ty = ry * RGY + tr;
    const bool tile_ok = tx < TXc && ty < TYc;
    const int tile = ty * TXc + tx;
    const int x0 = tx * CT, y0 = ty * CT;
    RunSmem& S = R[wid];
    int* const tp = P + wid * CAP;         // this tile's slices (tile-local ids in step 1)
    int* const tk = KY + wid * CAP;
    uint16_t* const tsz = SZ + wid * CAP;
    const uint32_t m = tile_ok && y0 + lane < f.H ? __ldg(rbits + (size_t)(y0 + lane) * f.bits_words + tx) : 0u;
    const uint32_t s = m & ~(m << 1);  // run starts
    const int nr = __popc(s);
    int rinc = nr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, rinc, o);
        if (lane >= o) rinc += v;
    }
    const int nruns = __shfl_sync(0xffffffffu, rinc, 31);
    if constexpr (FIRST) {
        if (threadIdx.x == 0) s_ovf = 0;
        __syncthreads();
        if (lane == 0 && nruns > CAP) s_ovf = 1;
        __syncthreads();
        if (s_ovf) {  // uniform: the whole region goes to the overflow pass
            if (threadIdx.x == 0) f.list[atomicAdd(&f.sc->n_ovf, 1u)] = (uint32_t)reg;
            return;
        }
    }
    S.rowm[lane] = m;
    S.rows[lane] = s;
    S.rs[lane] = rinc - nr;
    if (lane == 31) S.rs[CT] = rinc;
    {
        int k = rinc - nr;
        for (uint32_t t = s; t; t &= t - 1, ++k) {
            const int a = __ffs(t) - 1;
            S.rstart[k] = (uint8_t)a;
            S.rlen[k] = (uint8_t)run_len(m, a);
            S.rrow[k] = (uint8_t)lane;
        }
    }
    for (int i = lane; i < nruns; i += 32) {
        tp[i] = i;
        tsz[i] = 0;
    }
    __syncwarp();
    // 1. unions with the overlapping runs of the row above (8-connectivity).
    //   a. each run links to its FIRST overlapping run above (a smaller index:
    //      a forest whose roots are their trees' minima, no atomics);
    //   b. pointer jumping flattens it (in place: a concurrently updated
    //      par[par[i]] is still an ancestor; depth <= 32 rows -> 5 rounds);
    //   c. the remaining overlaps (merges: a run touching two or more runs
    //      above) are united with min-linking on the flattened forest, so
    //      the finds are short and a component's root stays its first run.
    auto overlaps = [&](int i, uint32_t& T, uint32_t& mu, uint32_t& su, int& r) {
        r = S.rrow[i];
        if (r == 0) return false;
        const int a = S.rstart[i], b = a + S.rlen[i] - 1;
        const int lo = a > 0 ? a - 1 : 0, hi = b < 31 ? b + 1 : 31;
        mu = S.rowm[r - 1];
        su = S.rows[r - 1];
        T = mu & upto_mask(hi) & ~((1u << lo) - 1u);
        return T != 0;
    };
    auto next_overlap = [&](uint32_t& T, uint32_t mu, uint32_t su, int r) {  // run index; T advanced
        const int j = __ffs(T) - 1;
        const uint32_t below = su & upto_mask(j);
        const int sa = 31 - __clz(below);
        const int e = sa + run_len(mu, sa) - 1;
        T &= e >= 31 ? 0u : ~upto_mask(e);
        return S.rs[r - 1] + __popc(below) - 1;
    };
    for (int i = lane; i < nruns; i += 32) {
        uint32_t T, mu, su;
        int r;
        tp[i] = overlaps(i, T, mu, su, r) ? next_overlap(T, mu, su, r) : i;
    }
    __syncwarp();
#pragma unroll 1
    for (int round = 0; round < 5; ++round) {
        for (int i = lane; i < nruns; i += 32) tp[i] = tp[tp[i]];
        __syncwarp();
    }
    for (int i = lane; i < nruns; i += 32) {
        uint32_t T, mu, su;
        int r;
        if (!overlaps(i, T, mu, su, r)) continue;
        next_overlap(T, mu, su, r);  // the first one: linked in (a)
        while (T) runite(tp, i, next_overlap(T, mu, su, r));
    }
    __syncwarp();
    // flatten, sizes at the tile-local roots; switch to region node ids
    auto gof = [&](const RunSmem& Q, int ri, int qx0, int qy0) { return (qy0 + Q.rrow[ri]) * f.W + qx0 + Q.rstart[ri]; };
    for (int i = lane; i < nruns; i += 32) {
        const int rt = rfind(tp, i);
        tp[i] = rt;
        sz_add(tsz, rt, S.rlen[i]);
    }
    __syncwarp();
    for (int i = lane; i < nruns; i += 32) {
        const int rt = tp[i];
        tk[i] = rt == i ? gof(S, i, x0, y0) : 0x7fffffff;
        tp[i] = wid * CAP + rt;
    }
    __syncthreads();
    // 2. inner borders of the region (the tile above / left, and the two
    //    upper diagonals), duplicates of a long border run skipped
    if (tr > 0) {
        const int wa = wid - RGX;
        const int a = node_at(R, wid, 0, lane);
        const int ap = __shfl_up_sync(0xffffffffu, a, 1);
        int u0 = lane > 0 ? node_at(R, wa, 31, lane - 1) : (tc > 0 ? node_at(R, wa - 1, 31, 31) : -1);
        int u1 = node_at(R, wa, 31, lane);
        int u2 = lane < 31 ? node_at(R, wa, 31, lane + 1) : (tc + 1 < RGX ? node_at(R, wa + 1, 31, 0) : -1);
        if (a >= 0) {
            const bool cont = lane > 0 && ap >= 0 && rfind(P, ap) == rfind(P, a);
            if (!cont && u0 >= 0) runite(P, a, u0);
            if (!cont && u1 >= 0) runite(P, a, u1);
            if (u2 >= 0) runite(P, a, u2);
        }
    }
    if (tc > 0) {
        const int wl = wid - 1;
        const int a = node_at(R, wid, lane, 0);
        if (a >= 0) {
            const int l0 = lane > 0 ? node_at(R, wl, lane - 1, 31) : -1;
            const int l1 = node_at(R, wl, lane, 31);
            const int l2 = lane < 31 ? node_at(R, wl, lane + 1, 31) : -1;
            if (l0 >= 0) runite(P, a, l0);
            if (l1 >= 0) runite(P, a, l1);
            if (l2 >= 0) runite(P, a, l2);
        }
    }
    __syncthreads();
    // region roots: key = min g, size = sum over their tile components
    for (int i = lane; i < nruns; i += 32) {
        const int self = wid * CAP + i;
        const int rt = rfind(P, self);
        if (tk[i] != 0x7fffffff && rt != self) {  // a tile root merged into another
            sz_add(SZ, rt, tsz[i]);
            atomicMin(&KY[rt], tk[i]);
        }
    }
    __syncthreads();
    // 3. region roots -> list; runs -> g; outer borders
    int nroots = 0;
    for (int i = lane; i < nruns; i += 32) {
        const int self = wid * CAP + i;
        nroots += rfind(P, self) == self;
    }
    int incl = nroots;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    unsigned base = 0;
    if (lane == 31 && incl) base = atomicAdd(&f.sc->n_lroots, (unsigned)incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    unsigned pos = base + incl - nroots;
    // region roots get dense ids (global union-find node = id: cpar, ccnt and
    // cmin = minimum raster index live in the first n_lroots entries of
    // f.par / f.cnt / f.roots, small enough to stay in L2)
    for (int i = lane; i < nruns; i += 32) {
        const int self = wid * CAP + i;
        if (rfind(P, self) == self) {
            const int id = (int)pos++;
            f.par[id] = id;
            f.cnt[id] = (uint32_t)tsz[i];
            f.roots[id] = tk[i];
            tk[i] = id;
        }
    }
    __syncthreads();
    auto gnode = [&](int node) {
        const int rt = rfind(P, node);
        return KY[rt];
    };
    if (tile_ok) {
        int32_t* rr = runroot + (size_t)tile * kRunCap;
        for (int i = lane; i < nruns; i += 32) rr[i] = gnode(wid * CAP + i);
    }
    int32_t* bd = bord + (size_t)reg * RBORD;
    if (tr == 0) {
        const int a = node_at(R, wid, 0, lane);
        bd[tc * CT + lane] = a >= 0 ? gnode(a) : -1;
    }
    if (tr == RGY - 1) {
        const int a = node_at(R, wid, 31, lane);
        bd[RW + tc * CT + lane] = a >= 0 ? gnode(a) : -1;
    }
    if (tc == 0) {
        const int a = node_at(R, wid, lane, 0);
        bd[2 * RW + tr * CT + lane] = a >= 0 ? gnode(a) : -1;
    }
    if (tc == RGX - 1) {
        const int a = node_at(R, wid, lane, 31);
        bd[2 * RW + RH + tr * CT + lane] = a >= 0 ? gnode(a) : -1;
    }
}

// B2 first pass: one CTA per region, 224-run tables with u16 sizes (105.6 KB
// of shared memory per 256x128 region: two CTAs per SM, so the 288 regions of
// a 4K frame run in one wave; dead-leaves masks peak at 224 runs per tile.
// 4 x 4 regions with 256-run tables: 45 us, 224-run: 38.7 us)
__global__ void __launch_bounds__(32 * NRW) k_ccl_region(Frame f, const uint32_t* __restrict__ rbits,
                                                         int32_t* __restrict__ runroot,
                                                         int32_t* __restrict__ bord) {
    extern __shared__ __align__(16) uint8_t smraw[];
    pdl_wait();
    {   // zero the size-histogram bins the prune will use (0..B+1)
        const unsigned long long B = budget_of(f);
        const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
        const long long stride = (long long)gridDim.x * blockDim.x;
        for (long long s = gt; s <= (long long)B + 1; s += stride) f.szhist[s] = 0;
        if (gt == 0) f.sc->budget = B;
    }
    ccl_region_body<kRunCapFast, true>(f, rbits, runroot, bord, blockIdx.x,
                                       smraw);
}

// B2 overflow pass: the regions the first pass listed (none on typical
// boundary masks), with the full 512-run tables
__global__ void __launch_bounds__(32 * NRW) k_ccl_region_ovf(Frame f, const uint32_t* __restrict__ rbits,
                                                             int32_t* __restrict__ runroot,
                                                             int32_t* __restrict__ bord) {
    extern __shared__ __align__(16) uint8_t smraw[];
    pdl_wait();
    const unsigned n = *(volatile unsigned*)&f.sc->n_ovf;
    for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
        ccl_region_body<kRunCap, false>(f, rbits, runroot, bord, (int)f.list[i], smraw);
        __syncthreads();  // the next region reuses the tables the last phase still reads
    }
}

bool pdl_on() {  // STK_PDL=0: plain launches in the boundary chain
    static const bool v = [] {
        const char* e = getenv("STK_PDL");
        return !e || atoi(e) != 0;
    }();
    return v;
}

template <typename... KArgs, typename... Args>
void launch_chain(void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t st, bool coop, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned na = 0;
    if (pdl_on()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, k, args...);
}

void launch_ccl_region(const Frame& f, const uint32_t* rbits, int32_t* runroot, int32_t* bord,
                       cudaStream_t st) {
    const int nreg = ((f.W + RW - 1) / RW) * ((f.H + RH - 1) / RH);
    const size_t s1 = region_smem_bytes<kRunCapFast>(), s2 = region_smem_bytes<kRunCap>();
    cudaFuncSetAttribute(k_ccl_region, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
    cudaFuncSetAttribute(k_ccl_region_ovf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
    launch_chain(k_ccl_region, dim3(nreg), dim3(32 * NRW), s1, st, false, f, rbits, runroot, bord);
    // a small grid: the pass is empty on typical masks (its launch is all it
    // costs), and each of its CTAs needs an SM's whole shared memory, so it
    // waits for SMs to drain while other frames run: 2 CTAs instead of 32,
    // +0.25 % frames/s (3 alternating runs)
    launch_chain(k_ccl_region_ovf, dim3(std::min(nreg, 2)), dim3(32 * NRW), s2, st, false, f, rbits, runroot, bord);
}

// ------------------------------------------------------------------ B3 ----
// Region outer borders: thread t < RW takes top-border pixel t (its three
// neighbours in the region above, corners from the regions above-left /
// above-right), thread RW + r the left-border pixel r (the left region's right
// column; the diagonals across region corners are covered by the top borders).
// A lane whose predecessor has the same root only adds its one new neighbour.
// With at most capn region roots (every frame-path mask seen: 6.5 K at 4K,
// 23 K at 8K) the unions are only listed (edges after the border labels in
// bord) and B3b unites them in shared memory; above it they run here on the
// global forest (lock-free, as B3b's fallback).
constexpr int kUniteThreads = 1024;

// the edge list: after the region border labels
__device__ __forceinline__ int2* edge_list(const Frame& f, int32_t* bord) {
    const int nreg = ((f.W + RW - 1) / RW) * ((f.H + RH - 1) / RH);
    return reinterpret_cast<int2*>(bord + (size_t)nreg * RBORD);
}

__global__ void __launch_bounds__(RW + RH) k_ccl_borders(Frame f, int32_t* __restrict__ bord, int capn,
                                                        uint32_t* __restrict__ sbits, int sbits_words) {
    __shared__ int s_wsum[(RW + RH) / 32];
    __shared__ unsigned s_base;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    pdl_wait();
    // the prune's size-s* bitmap is cleared here (no memset node in the chain)
    for (int i = blockIdx.x * (RW + RH) + t; i < sbits_words; i += gridDim.x * (RW + RH)) sbits[i] = 0u;
    const bool direct = (int)__ldcg(&f.sc->n_lroots) > capn;  // grid-uniform
    const int RXc = (f.W + RW - 1) / RW;
    const int reg = blockIdx.x;
    const int rx = reg % RXc, ry = reg / RXc;
    const int32_t* bd = bord + (size_t)reg * RBORD;
    int a, nb = 0, b[3] = {-1, -1, -1};
    if (t < RW) {
        a = ry > 0 ? bd[t] : -1;
        const int ap = __shfl_up_sync(0xffffffffu, a, 1);
        if (a >= 0) {
            const int32_t* up = bord + (size_t)(reg - RXc) * RBORD + RW;  // bottom row above
            const int u0 = t > 0 ? up[t - 1] : (rx > 0 ? bord[(size_t)(reg - RXc - 1) * RBORD + RW + RW - 1] : -1);
            const int u1 = up[t];
            const int u2 = t < RW - 1 ? up[t + 1] : (rx + 1 < RXc ? bord[(size_t)(reg - RXc + 1) * RBORD + RW] : -1);
            const bool cont = lane > 0 && ap == a;  // u0, u1 were the predecessor's u1, u2
            if (!cont && u0 >= 0) b[nb++] = u0;
            if (!cont && u1 >= 0 && u1 != u0) b[nb++] = u1;
            if (u2 >= 0 && u2 != u1) b[nb++] = u2;
        }
    } else {
        const int r = t - RW;
        a = rx > 0 ? bd[2 * RW + r] : -1;
        const int ap = __shfl_up_sync(0xffffffffu, a, 1);
        if (a >= 0) {
            const int32_t* lf = bord + (size_t)(reg - 1) * RBORD + 2 * RW + RH;  // right column, left
            const int l0 = r > 0 ? lf[r - 1] : -1;
            const int l1 = lf[r];
            const int l2 = r < RH - 1 ? lf[r + 1] : -1;
            const bool cont = lane > 0 && ap == a;
            if (!cont && l0 >= 0) b[nb++] = l0;
            if (!cont && l1 >= 0 && l1 != l0) b[nb++] = l1;
            if (l2 >= 0 && l2 != l1) b[nb++] = l2;
        }
    }
    if (direct) {
        if (nb) gunite_n(f.par, a, b, nb);
        return;
    }
    {   // a pair (a, b[i]) the previous lane also lists is dropped (along a
        // border run the same pair repeats lane after lane)
        const int ap = __shfl_up_sync(0xffffffffu, a, 1);
        const int p0 = __shfl_up_sync(0xffffffffu, b[0], 1);
        const int p1 = __shfl_up_sync(0xffffffffu, b[1], 1);
        const int p2 = __shfl_up_sync(0xffffffffu, b[2], 1);
        if (lane > 0 && ap == a) {
            int m = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
                if (i < nb && b[i] != p0 && b[i] != p1 && b[i] != p2) b[m++] = b[i];
            nb = m;
        }
    }
    // the block's edges appended with one atomic
    int incl = nb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (t == 0) {
        int tot = 0;
        for (int w = 0; w < (RW + RH) / 32; ++w) {
            const int v = s_wsum[w];
            s_wsum[w] = tot;
            tot += v;
        }
        s_base = tot ? atomicAdd(&f.sc->n_edges, (unsigned)tot) : 0u;
    }
    __syncthreads();
    int2* const el = edge_list(f, bord) + s_base + s_wsum[wid] + (incl - nb);
    for (int i = 0; i < nb; ++i) el[i] = make_int2(a, b[i]);
}

// B3b: one CTA unites the listed edges on a shared-memory forest of the n
// region roots (min-linking, path halving: shared-memory latency instead of
// the L2 round trips of global unions) and writes every non-root's final root
// to f.par (a flat forest: the later finds are one step).  Edges are read
// four per thread at a time so their L2 latencies overlap.  4K frame with
// 256x128 regions: 5411 roots, 9387 edges, ~20 us (B3's old global unions on
// 128x128 regions: 28 us).  Measured and dropped: hash-priority CAS linking
// (2.2x the union cycles), waves of one edge per thread with a flatten after
// each (1.5x), a converged lockstep walk with per-pair leader election (3x),
// lockstep walks of a thread's 8 roots, lanes of a warp on edges 32 apart
// (+17 %), an 8-CTA cluster with the forest in distributed shared memory
// (-5 %, not worth the cluster launch), shared-memory aggregation of the
// sizes (no change).
__global__ void __launch_bounds__(kUniteThreads, 1) k_ccl_unite(Frame f, const int32_t* __restrict__ bord, int capn,
                                                              int stats) {
    extern __shared__ int sp[];
    pdl_wait();
    const int n = (int)__ldcg(&f.sc->n_lroots);
    if (n > capn) return;  // B3 united them directly
    const int ne = (int)__ldcg(&f.sc->n_edges);
    const int2* el = edge_list(f, const_cast<int32_t*>(bord));
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += kUniteThreads) sp[i] = i;
    // stats with n <= PF threads' worth: the region roots' sizes and keys
    // fetched now, so their L2 latency hides behind the unions
    constexpr int PF = 8;
    const bool pf = stats && n <= PF * kUniteThreads;
    uint32_t pc[PF];
    int pk[PF];
    if (pf) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int i = tid + k * kUniteThreads;
            pc[k] = i < n ? __ldcg(f.cnt + i) : 0u;
            pk[k] = i < n ? __ldcg(f.roots + i) : 0;
        }
    }
    __syncthreads();
    constexpr int EB = 4;
    // a contiguous chunk of the list per thread: the lanes of a warp work on
    // 32 distant parts of the frame instead of one border's edges, which all
    // link the same region root (same-address atomics serialise)
    const int per = (ne + kUniteThreads - 1) / kUniteThreads;
    const int c0 = tid * per, c1 = min(c0 + per, ne);
    for (int e0 = c0; e0 < c1; e0 += EB) {
        int2 ed[EB];
#pragma unroll
        for (int j = 0; j < EB; ++j) ed[j] = e0 + j < c1 ? __ldcg(el + e0 + j) : make_int2(0, 0);
#pragma unroll
        for (int j = 0; j < EB; ++j) runite(sp, ed[j].x, ed[j].y);
    }
    __syncthreads();
    // stats (the prune path): the prune's B4 (sizes and minimum raster index
    // summed / min'ed at the roots) and B5 (root count, size histogram) here,
    // where the final roots are known, instead of two grid-barrier phases
    if (pf) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int i = tid + k * kUniteThreads;
            const int r = i < n ? rfind(sp, i) : i;
            if (r != i) {
                f.par[i] = r;
                atomicAdd(f.cnt + r, pc[k]);
                atomicMin(f.roots + r, pk[k]);
            }
        }
    } else {
        for (int i = tid; i < n; i += kUniteThreads) {
            const int r = rfind(sp, i);
            if (r != i) {
                f.par[i] = r;
                if (stats) {
                    atomicAdd(f.cnt + r, __ldcg(f.cnt + i));
                    atomicMin(f.roots + r, __ldcg(f.roots + i));
                }
            }
        }
    }
    if (!stats) return;
    __syncthreads();
    const unsigned long long B = __ldcg(&f.sc->budget);
    unsigned nr = 0;
    uint32_t sz[PF];  // with pf: the sizes of this thread's roots (0: not a root)
#pragma unroll
    for (int k = 0; k < PF; ++k) sz[k] = 0u;
    for (int i0 = tid; i0 < n; i0 += PF * kUniteThreads) {  // PF roots' sizes in flight at once
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int i = i0 + k * kUniteThreads;
            sz[k] = i < n && sp[i] == i ? __ldcg(f.cnt + i) : 0u;  // roots: unchanged since the unions
        }
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            if (sz[k] == 0) continue;  // non-roots (a root holds >= 1 pixel)
            ++nr;
            // with pf the global size histogram is only needed if the select
            // below falls back to the cooperative prune (hist_out)
            if (!pf && sz[k] <= B + 1) atomicAdd(f.szhist + sz[k], 1u);
        }
    }
    auto hist_out = [&]() {
#pragma unroll
        for (int k = 0; k < PF; ++k)
            if (sz[k] != 0 && sz[k] <= B + 1) atomicAdd(f.szhist + sz[k], 1u);
    };
    nr = __reduce_add_sync(0xffffffffu, nr);
    if ((tid & 31) == 0 && nr) atomicAdd(&f.sc->n_roots, nr);
    if (tid == 0) f.sc->united = 1u;
    // B6 + B7 here too when s* <= SB and at most LCAP components have size s*
    // (every frame-path mask seen): the cooperative prune then has nothing
    // left and returns at once.  Same rule as its phases: s* = the smallest
    // size whose class-cumulative pixel count CS(s*) exceeds B (B + 2 when
    // CS(B + 1) <= B), q = (B - CS(s* - 1)) / s*; sizes < s* removed and the
    // q size-s* components with the smallest raster keys.
    constexpr int SB = 4096, LCAP = 2048;
    if (!pf) return;
    if (n + SB + 2 * LCAP > capn) {  // block-uniform
        hist_out();
        return;
    }
    int* const hist = sp + n;  // hist[s - 1], s = 1..SB
    int* const lkey = hist + SB;
    int* const lid = lkey + LCAP;
    __shared__ unsigned long long s_wtot[kUniteThreads / 32];
    __shared__ unsigned long long s_q;
    __shared__ int s_star, s_cnt;
    const long long L = min((long long)B + 1, (long long)SB);
    for (int i = tid; i < SB; i += kUniteThreads) hist[i] = 0;
    if (tid == 0) {
        s_star = -1;
        s_cnt = 0;
        s_q = 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PF; ++k)
        if (sz[k] != 0 && (long long)sz[k] <= L) atomicAdd(&hist[sz[k] - 1], 1);
    __syncthreads();
    static_assert(SB == 4 * kUniteThreads, "four bins per thread");
    unsigned long long v[4], tsum = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const long long sv = 4 * tid + j + 1;
        v[j] = sv <= L ? (unsigned long long)sv * (unsigned)hist[sv - 1] : 0ull;
        tsum += v[j];
    }
    {   // exclusive block scan of tsum
        const int lane = tid & 31, wid = tid >> 5;
        unsigned long long x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wtot[wid] = x;
        __syncthreads();
        unsigned long long off = 0;
        for (int w = 0; w < wid; ++w) off += s_wtot[w];
        unsigned long long cs = off + x - tsum;  // CS(4 tid)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (cs <= B && cs + v[j] > B) {  // the first crossing (CS is non-decreasing)
                s_star = 4 * tid + j + 1;
                s_q = (B - cs) / (unsigned long long)(4 * tid + j + 1);
            }
            cs += v[j];
        }
    }
    __syncthreads();
    long long sst = s_star;
    const unsigned long long q = s_q;
    if (sst < 0) {
        if (L < (long long)B + 1) {  // s* > SB: the cooperative prune decides
            hist_out();
            return;
        }
        sst = (long long)B + 2;             // CS(B + 1) <= B: every size <= B + 1 goes
    }
    // the size-s* class (q > 0): listed first, so an over-long list falls back
    // before anything is written
    if (q > 0) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            if (sz[k] != sst) continue;
            const int i = tid + k * kUniteThreads;
            const int at = atomicAdd(&s_cnt, 1);
            if (at < LCAP) {
                lkey[at] = __ldcg(f.roots + i);
                lid[at] = i;
            }
        }
        __syncthreads();
        if (s_cnt > LCAP) {  // block-uniform
            hist_out();
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < PF; ++k)
        if (sz[k] != 0 && (long long)sz[k] < sst) f.cnt[tid + k * kUniteThreads] = sz[k] | kRemoved;
    if (q > 0) {
        const int c = s_cnt;
        for (int e = tid; e < c; e += kUniteThreads) {  // rank by key (keys are distinct raster indices)
            const int ke = lkey[e];
            int r = 0;
            for (int j = 0; j < c; ++j) r += lkey[j] < ke;
            if ((unsigned long long)r < q) f.cnt[lid[e]] = (uint32_t)sst | kRemoved;
        }
    }
    if (tid == 0) {
        f.sc->s_star = (unsigned long long)sst;
        f.sc->q = q;
        f.sc->pruned = 1u;
    }
}

// 256-thread exclusive block scan (u64) used by the prune select.

__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* sh,
                                                              unsigned long long* total) {
    // 256 threads
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    unsigned long long off = 0, tot = 0;
    for (int i = 0; i < 8; ++i) {
        if (i < wid) off += sh[i];
        tot += sh[i];
    }
    __syncthreads();
    *total = tot;
    return off + x - v;
}

// ------------------------------------------------------------------ B8 ----
__global__ void __launch_bounds__(128) k_apply_runs(Frame f, const uint32_t* __restrict__ rbits,
                                                    const int32_t* __restrict__ runroot, int anchors) {
    __shared__ unsigned long long red[3][4];
    pdl_wait();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TXc = (f.W + CT - 1) / CT, TYc = (f.H + CT - 1) / CT;
    const int tile = blockIdx.x * 4 + wid;
    unsigned long long kept = 0, matched = 0, ops = 0;
    if (tile < TXc * TYc) {
        const int tx = tile % TXc, x0 = tx * CT, y0 = (tile / TXc) * CT;
        const int y = y0 + lane;
        const bool rowok = y < f.H;
        const uint32_t m = rowok ? __ldg(rbits + (size_t)y * f.bits_words + tx) : 0u;
        const uint32_t s = m & ~(m << 1);
        const int nr = __popc(s);
        int rinc = nr;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, rinc, o);
            if (lane >= o) rinc += v;
        }
        const int32_t* rr = runroot + (size_t)tile * kRunCap + (rinc - nr);
        uint32_t pruned = 0;
        // run -> region root id -> global root -> removed?  Three dependent L2
        // reads per run: issued for up to 8 runs of the row at a time (one
        // latency exposure per level instead of one per run)
        constexpr int RB = 8;
        uint32_t t = s;
        for (int k0 = 0; k0 < nr; k0 += RB) {
            int id[RB], rt[RB];
            uint32_t cn[RB];
#pragma unroll
            for (int k = 0; k < RB; ++k) id[k] = k0 + k < nr ? __ldg(rr + k0 + k) : 0;
#pragma unroll
            for (int k = 0; k < RB; ++k) rt[k] = k0 + k < nr ? __ldcg(f.par + id[k]) : 0;
#pragma unroll
            for (int k = 0; k < RB; ++k) cn[k] = k0 + k < nr ? __ldcg(f.cnt + rt[k]) : kRemoved;
#pragma unroll
            for (int k = 0; k < RB; ++k) {
                if (k0 + k < nr) {
                    const int a = __ffs(t) - 1, len = run_len(m, a);
                    t &= t - 1;
                    if (!(cn[k] & kRemoved)) pruned |= (len >= 32 ? 0xffffffffu : ((1u << len) - 1u)) << a;
                }
            }
        }
        const int mg = f.hw, W = f.W, H = f.H;
        uint32_t anc = pruned;
        if (anchors && rowok && y >= mg && y <= H - 1 - mg) {
            if (mg >= x0 && mg < x0 + 32) anc |= 1u << (mg - x0);
            const int xr = W - 1 - mg;
            if (xr >= x0 && xr < x0 + 32) anc |= 1u << (xr - x0);
        }
        // matchable: anchored and the window fits (h <= x < W-h, h <= y < H-h)
        uint32_t mat = 0;
        if (rowok && y >= mg && y < H - mg) {
            const int lo = max(mg - x0, 0), hi = min(W - mg - x0, 32);  // [lo, hi)
            if (hi > lo) {
                const uint32_t win = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
                mat = anc & win;
            }
        }
        if (rowok) {
            f.mbits[(size_t)y * f.bits_words + tx] = mat;
            if (tx == TXc - 1)  // row-tile padding words read by the strip SAD kernel
                for (int wd = tx + 1; wd < f.bits_words; ++wd) f.mbits[(size_t)y * f.bits_words + wd] = 0u;
            if (f.mprn) {
                store_bits_as_bytes(f.mprn + (size_t)y * f.P + x0, pruned);
                store_bits_as_bytes(f.manc + (size_t)y * f.P + x0, anc);
            }
        }
        kept = __popc(pruned);
        matched = __popc(mat);
        if (mat) {
            // sum over matchable pixels of min(D, x - h) + 1
            if (x0 - mg >= f.D) {
                ops = (unsigned long long)matched * (f.D + 1);
            } else {
                for (uint32_t t = mat; t; t &= t - 1) ops += min(f.D, x0 + __ffs(t) - 1 - mg) + 1;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        kept += __shfl_xor_sync(0xffffffffu, kept, o);
        matched += __shfl_xor_sync(0xffffffffu, matched, o);
        ops += __shfl_xor_sync(0xffffffffu, ops, o);
    }
    if (lane == 0) {
        red[0][wid] = kept;
        red[1][wid] = matched;
        red[2][wid] = ops;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long a = red[0][0] + red[0][1] + red[0][2] + red[0][3];
        const unsigned long long b = red[1][0] + red[1][1] + red[1][2] + red[1][3];
        const unsigned long long c = red[2][0] + red[2][1] + red[2][2] + red[2][3];
        if (a) atomicAdd(&f.sc->pruned_count, a);
        if (b) {
            atomicAdd(&f.sc->matched, b);
            atomicAdd(&f.sc->n_list, (unsigned)b);
        }
        if (c) atomicAdd(&f.sc->sad_ops, c * (unsigned long long)(f.window * f.window));
    }
}

// ------------------------------------------------------------------ B9 ----
// Raster-ordered list of matchable pixels + per-row-tile offsets from the
// matchable bits (the per-pixel list SAD kernel's input).  Chunk = 32 row-tiles
// of 128 pixels = 128 words; single-pass decoupled look-back.
__global__ void __launch_bounds__(128) k_list_bits(Frame f) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[4];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* status = f.lb + LB_LIST * f.lb_stride;
    if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_LIST], 1u);
    __syncthreads();
    const int c = (int)s_chunk;
    // thread -> one row-tile (4 words) of the chunk
    const int t = c * kTilesPerChunk + threadIdx.x;
    const bool tv = threadIdx.x < kTilesPerChunk && t < f.n_tiles;
    uint32_t w[4] = {0, 0, 0, 0}, cnt = 0;
    int y = 0, seg = 0;
    if (tv) {
        y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            w[j] = f.mbits[(size_t)y * f.bits_words + seg * 4 + j];
            cnt += __popc(w[j]);
        }
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wcount[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t agg = __reduce_add_sync(0xffffffffu, lane < 4 ? wcount[lane] : 0u);
        const uint32_t excl = lb_exclusive_warp(status, c, agg);
        if (lane == 0) {
            s_excl = excl;
            if (c == f.n_chunks - 1) f.tile_off[f.n_tiles] = excl + agg;
        }
    }
    __syncthreads();
    if (!tv) return;
    uint32_t pos = s_excl + incl - cnt;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    f.tile_off[t] = pos;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        for (uint32_t b = w[j]; b; b &= b - 1) {
            const int x = seg * kRowTile + j * 32 + __ffs(b) - 1;
            f.list[pos++] = ((uint32_t)y << 16) | (uint32_t)x;
        }
}

// ------------------------------------------------------------- B4-B7 fused --
// One cooperative launch (all blocks co-resident) runs compress, root stats,
// the s*/q select, the size classes and the first-q raster scan, separated by
// grid barriers instead of five kernel boundaries.
__device__ __forceinline__ void grid_barrier(DevScalars* sc, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = &sc->gbar_gen;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(&sc->gbar_count, 1u) == nblocks - 1) {
            sc->gbar_count = 0;
            __threadfence();
            atomicAdd(&sc->gbar_gen, 1u);
        } else {
            while (*vgen == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_prune_fused(Frame f, uint32_t* __restrict__ sbits,
                                                     int nwords) {
    __shared__ unsigned long long sh[8];
    __shared__ int s_blk;
    __shared__ unsigned long long s_before;
    __shared__ uint32_t s_wsum[8];
    pdl_wait();
    DevScalars* sc = f.sc;
    if (__ldcg(&sc->pruned)) return;  // grid-uniform: B3b did B6 + B7
    const unsigned G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int gt = blockIdx.x * 256 + tid, gs = G * 256;
    const int n = (int)sc->n_lroots;
    const unsigned long long B = sc->budget;
    // B4, B5: done by B3b unless B3 united on the global forest (grid-uniform)
    if (!__ldcg(&sc->united)) {
        // B4 compress
        for (int id = gt; id < n; id += gs) {
            const int r = gfind_ro(f.par, id);
            if (r != id) {
                f.par[id] = r;
                atomicAdd(f.cnt + r, __ldcg(f.cnt + id));
                atomicMin(f.roots + r, __ldcg(f.roots + id));
            }
        }
        grid_barrier(sc, G);
        // B5 root stats
        {
            unsigned nr = 0;
            for (int id = gt; id < n; id += gs) {
                if (__ldcg(f.par + id) == id) {
                    ++nr;
                    const uint32_t sz = __ldcg(f.cnt + id);
                    if (sz <= B + 1) atomicAdd(f.szhist + sz, 1u);
                }
            }
            nr = __reduce_add_sync(0xffffffffu, nr);
            if (lane == 0 && nr) atomicAdd(&sc->n_roots, nr);
        }
        grid_barrier(sc, G);
    }
    // B6 select: block sums over sizes 1..B+1, then block 0 finds s*, q
    const long long L = (long long)B + 1;
    const long long per = (L + G - 1) / G;
    auto bin_sum = [&](long long a0, long long a1) {
        const long long pt = (a1 - a0 + 255) / 256;
        const long long t0 = a0 + tid * pt, t1 = min(t0 + pt, a1);
        unsigned long long sum = 0;
        for (long long s = t0; s < t1; ++s) sum += (unsigned long long)s * __ldcg(f.szhist + s);
        return sum;
    };
    {
        const long long a0 = 1 + blockIdx.x * per, a1 = min(a0 + per, L + 1);
        unsigned long long tot;
        block_excl_scan(a0 < a1 ? bin_sum(a0, a1) : 0ull, sh, &tot);
        if (tid == 0) sc->gsum[blockIdx.x] = tot;
    }
    grid_barrier(sc, G);
    if (blockIdx.x == 0) {
        if (tid == 0) {
            sc->s_star = B + 2;
            sc->q = 0;
            s_blk = -1;
        }
        // scan the G block sums (G <= 256 * ... handled in chunks of 256)
        unsigned long long base = 0;
        for (int c0 = 0; c0 < (int)G; c0 += 256) {
            const int i = c0 + tid;
            const unsigned long long v = i < (int)G ? __ldcg(&sc->gsum[i]) : 0ull;
            unsigned long long tot;
            const unsigned long long before = base + block_excl_scan(v, sh, &tot);
            if (i < (int)G && before <= B && before + v > B) {
                s_blk = i;
                s_before = before;
            }
            base += tot;
        }
        __syncthreads();
        if (s_blk >= 0) {
            const long long a0 = 1 + s_blk * per, a1 = min(a0 + per, L + 1);
            const long long pt = (a1 - a0 + 255) / 256;
            const long long t0 = a0 + tid * pt, t1 = min(t0 + pt, a1);
            unsigned long long mine = 0;
            for (long long s = t0; s < t1; ++s) mine += (unsigned long long)s * __ldcg(f.szhist + s);
            unsigned long long tot;
            const unsigned long long tb = s_before + block_excl_scan(mine, sh, &tot);
            if (tb <= B && tb + mine > B) {
                unsigned long long cs = tb;
                for (long long s = t0; s < t1; ++s) {
                    const unsigned long long add = (unsigned long long)s * __ldcg(f.szhist + s);
                    if (cs + add > B) {
                        sc->s_star = (unsigned long long)s;
                        sc->q = (B - cs) / (unsigned long long)s;
                        break;
                    }
                    cs += add;
                }
            }
        }
    }
    grid_barrier(sc, G);
    // B7 size classes
    const unsigned long long sst = sc->s_star, q = sc->q;
    for (int id = gt; id < n; id += gs) {
        if (__ldcg(f.par + id) != id) continue;
        const uint32_t sz = __ldcg(f.cnt + id);
        if (sz < sst) {
            f.cnt[id] = sz | kRemoved;
        } else if (sz == sst && q > 0) {
            const int k = __ldcg(f.roots + id);
            f.rank[k] = id;
            atomicOr(sbits + (k >> 5), 1u << (k & 31));
        }
    }
    if (q == 0) return;  // uniform: no barrier is pending
    grid_barrier(sc, G);
    // B7b: the first q size-s* components in raster order.  Block b owns words
    // [b * per_w, (b + 1) * per_w); counts, barrier, prefix over earlier blocks.
    const int per_w = (nwords + G - 1) / G;
    const int w0 = blockIdx.x * per_w, w1 = min(w0 + per_w, nwords);
    uint32_t mycnt = 0;
    for (int i = w0 + tid; i < w1; i += 256) mycnt += __popc(__ldcg(sbits + i));
    mycnt = __reduce_add_sync(0xffffffffu, mycnt);
    if (lane == 0) s_wsum[wid] = mycnt;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int i = 0; i < 8; ++i) t += s_wsum[i];
        sc->gcnt[blockIdx.x] = t;
    }
    grid_barrier(sc, G);
    uint32_t before = 0;
    for (int i = tid; i < (int)blockIdx.x; i += 256) before += __ldcg(&sc->gcnt[i]);
    before = __reduce_add_sync(0xffffffffu, before);
    if (lane == 0) s_wsum[wid] = before;
    __syncthreads();
    uint32_t run = 0;
    for (int i = 0; i < 8; ++i) run += s_wsum[i];
    if (run >= q) return;
    // walk the block's words in order, 256 at a time, warp-then-block scan
    for (int c0 = w0; c0 < w1 && run < q; c0 += 256) {
        const int i = c0 + tid;
        const uint32_t wd = i < w1 ? __ldcg(sbits + i) : 0u;
        const uint32_t cnt = __popc(wd);
        unsigned long long tot;
        const uint32_t ex = (uint32_t)block_excl_scan(cnt, sh, &tot);
        uint32_t rk = run + ex;
        for (uint32_t t = wd; t && rk < q; t &= t - 1, ++rk) {
            const int k = i * 32 + __ffs(t) - 1;
            f.cnt[__ldcg(f.rank + k)] |= kRemoved;
        }
        run += (uint32_t)tot;
    }
}

// Stage entry prune_components: a byte mask (pitched) -> bit rows + count.
__global__ void __launch_bounds__(256) k_mask_to_bits(Frame f, const uint8_t* __restrict__ mask,
                                                      uint32_t* __restrict__ rbits) {
    const int BW = (f.W + 31) / 32;
    const long long nw = (long long)BW * f.H;
    unsigned long long cnt = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nw;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / BW), wc = (int)(i - (long long)y * BW);
        const uint8_t* row = mask + (size_t)y * f.P + 32 * wc;
        uint32_t m = 0;
        for (int b = 0; b < 32 && 32 * wc + b < f.W; ++b) m |= (row[b] ? 1u : 0u) << b;
        rbits[(size_t)y * f.bits_words + wc] = m;
        cnt += __popc(m);
    }
    cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&f.sc->refined_count, cnt);
}

}  // namespace

size_t bord_bytes(int W, int H) {  // the border labels of every region (B2 -> B3) + B3's edges
    const size_t nreg = (size_t)((W + RW - 1) / RW) * ((H + RH - 1) / RH);
    return nreg * RBORD * sizeof(int32_t) + nreg * (RW + RH) * 3 * sizeof(int2);
}

// B3 + B3b.  capn: the most region roots B3b's shared-memory forest takes
// (STK_UNITE_CAP: test / experiment knob; 0 forces the global unions)
// sbits (prune path): cleared by B3 for B4-B7
int launch_ccl_borders(const Frame& f, int32_t* bord, bool stats, uint32_t* sbits, int sbits_words,
                       cudaStream_t st) {  // kernels launched
    static const int capn = [] {
        const char* e = getenv("STK_UNITE_CAP");
        return e ? atoi(e) : 32768;
    }();
    const int nreg = ((f.W + RW - 1) / RW) * ((f.H + RH - 1) / RH);
    launch_chain(k_ccl_borders, dim3(nreg), dim3(RW + RH), 0, st, false, f, bord, capn, sbits,
                 sbits ? sbits_words : 0);
    if (capn > 0) {
        const int smem = capn * (int)sizeof(int);
        cudaFuncSetAttribute(k_ccl_unite, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        launch_chain(k_ccl_unite, dim3(1), dim3(kUniteThreads), (size_t)smem, st, false, f, (const int32_t*)bord, capn,
                     stats ? 1 : 0);
        return 2;
    }
    return 1;
}

int launch_ccl_prune_bits(const Frame& f, uint32_t* rbits, int32_t* runroot, int32_t* bord,
                           uint32_t* sbits, int sbits_words, bool anchors, cudaStream_t st) {
    // B2 - B8
    const int ntiles = ((f.W + CT - 1) / CT) * ((f.H + CT - 1) / CT);
    const int tb = (ntiles + 3) / 4;
    launch_ccl_region(f, rbits, runroot, bord, st);  // 2 kernels
    const int nb = launch_ccl_borders(f, bord, true, sbits, sbits_words, st);
    {   // B4-B7 in one cooperative launch (co-resident blocks, grid barriers)
        // co-resident blocks per SM depend only on the kernel (thread-safe
        // static init); the grid follows the context's device SM count
        static const int per_sm = [] {
            int n = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_prune_fused, 256, 0);
            return n;
        }();
        // one block per SM (STK_PRUNE_BPS: experiment knob): blocks spinning at
        // the grid barriers hold SMs that other frames' kernels could use
        // (4K frame period 0.665 -> 0.659 ms vs two per SM)
        static const int bps = [] {
            const char* e = getenv("STK_PRUNE_BPS");
            return e ? atoi(e) : 1;
        }();
        // the phases are short loops between grid barriers and the blocks mostly
        // wait: fewer blocks than SMs leave the others to other frames' kernels.
        // One block per 2^17 pixels (>= 8; 72 at 4K): 1605 -> 1642 frames/s vs
        // one per SM with the stage's own time unchanged (0.155 ms; 2^19: 18
        // blocks, same frames/s, 0.163-0.181 ms).  STK_PRUNE_SHIFT: experiment knob.
        static const int pshift = [] {
            const char* e = getenv("STK_PRUNE_SHIFT");
            return e ? atoi(e) : 17;
        }();
        int g_blocks = std::min(512, std::max(1, std::min(per_sm, bps)) * f.sms);  // <= gsum/gcnt slots
        g_blocks = std::min<long long>(g_blocks, std::max<long long>(8, (f.N + (1ll << pshift) - 1) >> pshift));
        launch_chain(k_prune_fused, dim3(g_blocks), dim3(256), 0, st, true, f, sbits, (int)sbits_words);
    }
    launch_chain(k_apply_runs, dim3(tb), dim3(128), 0, st, false, f, (const uint32_t*)rbits, (const int32_t*)runroot,
                 anchors ? 1 : 0);
    return 2 + nb + 2;  // B2 (+ overflow pass), B3 (+ B3b), B4-B7, B8
}

void launch_prune_mask_bits(const Frame& f, const uint8_t* mask, uint32_t* rbits, int32_t* runroot,
                            int32_t* bord, uint32_t* sbits, int sbits_words, cudaStream_t st) {
    if (f.N == 0) return;
    const long long nw = (long long)((f.W + 31) / 32) * f.H;
    k_mask_to_bits<<<(int)std::min<long long>((nw + 255) / 256, f.sms * 8), 256, 0, st>>>(f, mask, rbits);
    launch_ccl_prune_bits(f, rbits, runroot, bord, sbits, sbits_words, false, st);
}

int launch_boundary_bits(const Frame& f, uint32_t* rbits, int32_t* runroot, int32_t* bord,
                         uint32_t* sbits, int sbits_words, bool anchors, bool want_list,
                         cudaStream_t st) {
    if (f.N == 0) return 0;
    // B1
    const int BW = (f.W + 31) / 32;
    const int strips = (BW + MB_WPW - 1) / MB_WPW, bands = (f.H + MB_ROWS - 1) / MB_ROWS;
    const int warps = strips * bands;
    int npl = 1;
    while ((1 << npl) < f.kcfg && npl < 8) ++npl;
    const int gb = (warps + 3) / 4;
    switch (npl) {
        case 1: k_morph_bits<1, MB_FRAME><<<gb, 128, 0, st>>>(f, rbits, nullptr, 0); break;
        case 2: k_morph_bits<2, MB_FRAME><<<gb, 128, 0, st>>>(f, rbits, nullptr, 0); break;
        case 3: k_morph_bits<3, MB_FRAME><<<gb, 128, 0, st>>>(f, rbits, nullptr, 0); break;
        case 4: k_morph_bits<4, MB_FRAME><<<gb, 128, 0, st>>>(f, rbits, nullptr, 0); break;
        default: k_morph_bits<8, MB_FRAME><<<gb, 128, 0, st>>>(f, rbits, nullptr, 0); break;
    }
    int n = 1 + launch_ccl_prune_bits(f, rbits, runroot, bord, sbits, sbits_words, anchors, st);
    if (want_list) {
        k_list_bits<<<f.n_chunks, 128, 0, st>>>(f);
        ++n;
    }
    return n;
}

// Stage entries detect_boundaries / morph_fill / morph_remove on B1 (the frame
// path's word-parallel morphology), then bits -> the reference's bytes.
// mode: 1 detect (src = u16 labels, pitch 2P), 2 fill, 3 remove (src = byte
// mask, pitch P); out = pitched bytes.
void launch_morph_stage_bits(const Frame& f, int mode, const uint8_t* src, uint32_t* rbits,
                             uint8_t* out, cudaStream_t st) {
    if (f.N == 0) return;
    const int BW = (f.W + 31) / 32;
    const int strips = (BW + MB_WPW - 1) / MB_WPW, bands = (f.H + MB_ROWS - 1) / MB_ROWS;
    const int gb = (strips * bands + 3) / 4;
    const long long nw = (long long)BW * f.H;
    const int cb = (int)std::min<long long>((nw + 255) / 256, f.sms * 8);
    if (mode == MB_DET16) {
        k_morph_bits<8, MB_DET16><<<gb, 128, 0, st>>>(f, rbits, src, 0);  // label bits 0..7
        k_morph_bits<8, MB_DET16><<<gb, 128, 0, st>>>(f, rbits, src, 8);  // label bits 8..15
        k_bits_to_bytes<MB_DET16><<<cb, 256, 0, st>>>(f, rbits, nullptr, out);
    } else if (mode == MB_FILL) {
        k_morph_bits<1, MB_FILL><<<gb, 128, 0, st>>>(f, rbits, src, 0);
        k_bits_to_bytes<MB_FILL><<<cb, 256, 0, st>>>(f, rbits, src, out);
    } else {
        k_morph_bits<1, MB_REMOVE><<<gb, 128, 0, st>>>(f, rbits, src, 0);
        k_bits_to_bytes<MB_REMOVE><<<cb, 256, 0, st>>>(f, rbits, src, out);
    }
}

// ------------------------------------------------ label_components ------
// The stage entry label_components (boundary.cpp:87-148) on the frame path's
// run CCL (B2/B3): the reference's label of a component is the rank, in raster
// order, of its first pixel (its minimum raster index g, which B2/B4 keep at
// every root).  L1 compresses the region-root forest (as B4); L2 marks g of
// every root in a raster bitmap and counts roots; the bitmap's word popcounts
// are scanned (cub, in place); L3 gives each root label = rank(g) = word
// offset + popcount below g, sizes[label], ids[label] = label; L4 writes the
// per-pixel labels from the runs (-1 on unset pixels).
namespace {

__global__ void __launch_bounds__(256) k_cc_compress(Frame f) {
    const int n = (int)f.sc->n_lroots;
    for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
        const int r = gfind_ro(f.par, id);
        if (r != id) {
            f.par[id] = r;
            atomicAdd(f.cnt + r, __ldcg(f.cnt + id));
            atomicMin(f.roots + r, __ldcg(f.roots + id));
        }
    }
}

__global__ void __launch_bounds__(256) k_cc_mark(Frame f, uint32_t* __restrict__ gbits) {
    const int n = (int)f.sc->n_lroots;
    unsigned nr = 0;
    for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
        if (__ldcg(f.par + id) == id) {
            const int g = __ldcg(f.roots + id);
            atomicOr(gbits + (g >> 5), 1u << (g & 31));
            ++nr;
        }
    }
    nr = __reduce_add_sync(0xffffffffu, nr);
    if ((threadIdx.x & 31) == 0 && nr) atomicAdd(&f.sc->n_roots, nr);
}

__global__ void __launch_bounds__(256) k_cc_popc(const uint32_t* __restrict__ gbits, uint32_t* __restrict__ wcnt,
                                                 int nw) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += gridDim.x * blockDim.x)
        wcnt[i] = __popc(gbits[i]);
}

__global__ void __launch_bounds__(256) k_cc_root_labels(Frame f, const uint32_t* __restrict__ gbits,
                                                        const uint32_t* __restrict__ woff,
                                                        uint32_t* __restrict__ sizes, int32_t* __restrict__ ids) {
    const int n = (int)f.sc->n_lroots;
    for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < n; id += gridDim.x * blockDim.x) {
        if (__ldcg(f.par + id) != id) continue;
        const int g = __ldcg(f.roots + id);
        const int label = (int)(woff[g >> 5] + __popc(gbits[g >> 5] & ((1u << (g & 31)) - 1u)));
        f.rank[id] = label;
        sizes[label] = __ldcg(f.cnt + id);
        ids[label] = label;
    }
}

__global__ void __launch_bounds__(128) k_cc_write_labels(Frame f, const uint32_t* __restrict__ rbits,
                                                         const int32_t* __restrict__ runroot,
                                                         int32_t* __restrict__ labels) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int TXc = (f.W + CT - 1) / CT, TYc = (f.H + CT - 1) / CT;
    const int tile = blockIdx.x * 4 + wid;
    if (tile >= TXc * TYc) return;
    const int tx = tile % TXc, x0 = tx * CT, y = (tile / TXc) * CT + lane;
    const uint32_t m = y < f.H ? __ldg(rbits + (size_t)y * f.bits_words + tx) : 0u;
    const uint32_t s = m & ~(m << 1);
    const int nr = __popc(s);
    int rinc = nr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, rinc, o);
        if (lane >= o) rinc += v;
    }
    if (y >= f.H) return;
    const int32_t* rr = runroot + (size_t)tile * kRunCap + (rinc - nr);
    int32_t* out = labels + (size_t)y * f.W + x0;
    const int nx = min(CT, f.W - x0);
    int k = 0, x = 0;
    for (uint32_t t = s; t; t &= t - 1, ++k) {
        const int a = __ffs(t) - 1, len = run_len(m, a);
        const int lab = __ldcg(f.rank + __ldcg(f.par + __ldg(rr + k)));
        for (; x < a; ++x) out[x] = -1;
        for (; x < a + len; ++x) out[x] = lab;
    }
    for (; x < nx; ++x) out[x] = -1;
}

}  // namespace

// mask (pitched bytes) -> labels (dense i32, -1 unset), sizes[C], ids[C] =
// 0..C-1 (the caller sorts them into by_size); C in f.sc->n_roots.  gbits:
// N/32-word raster bitmap, wscan: >= N/32 + 1 words, tmp/tmp_bytes: cub.
void launch_label_components_bits(const Frame& f, const uint8_t* mask, uint32_t* rbits, int32_t* runroot,
                                  int32_t* bord, uint32_t* gbits, int gbits_words, uint32_t* wscan,
                                  void* tmp, size_t tmp_bytes, int32_t* labels, uint32_t* sizes,
                                  int32_t* ids, cudaStream_t st) {
    if (f.N == 0) return;
    const long long nw = (long long)((f.W + 31) / 32) * f.H;
    const int gb = (int)std::min<long long>((nw + 255) / 256, f.sms * 8);
    k_mask_to_bits<<<gb, 256, 0, st>>>(f, mask, rbits);
    launch_ccl_region(f, rbits, runroot, bord, st);  // B2
    launch_ccl_borders(f, bord, false, nullptr, 0, st);  // B3, B3b (k_cc_compress aggregates)
    const int ib = f.sms * 4;
    k_cc_compress<<<ib, 256, 0, st>>>(f);
    cudaMemsetAsync(gbits, 0, (size_t)gbits_words * 4, st);
    k_cc_mark<<<ib, 256, 0, st>>>(f, gbits);
    k_cc_popc<<<(gbits_words + 255) / 256, 256, 0, st>>>(gbits, wscan, gbits_words);
    size_t need = tmp_bytes;
    cub::DeviceScan::ExclusiveSum(tmp, need, wscan, wscan, gbits_words, st);  // in place
    k_cc_root_labels<<<ib, 256, 0, st>>>(f, gbits, wscan, sizes, ids);
    const int ntiles = ((f.W + CT - 1) / CT) * ((f.H + CT - 1) / CT);
    k_cc_write_labels<<<(ntiles + 3) / 4, 128, 0, st>>>(f, rbits, runroot, labels);
}

size_t label_components_tmp_bytes(int gbits_words) {
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, (uint32_t*)nullptr, (uint32_t*)nullptr, gbits_words);
    return need;
}

}  // namespace stk
