// K5c sad_ws -- warp-specialised column-sum SAD matching (default SAD kernel).
//
// Same arithmetic as K5b (integer sums are associative, so sliding column and
// window sums give exactly the cost of the reference's per-pixel loop,
// stereo.cpp:12-28, and therefore the same winner, stereo.cpp:90-97), with
// the work split into two warp roles that run concurrently inside one CTA
// instead of alternating behind __syncthreads():
//
//   staging   the band's rows of both gray views stream through a ring of RS
//             row slots with 1-D bulk TMA (cp.async.bulk, UBLKCP) and a full
//             mbarrier per slot; vertical thread 0 refills a slot as soon as
//             the EMPTY hand-off below proves every vertical thread is past it.
//   vertical  (NVW warps) thread = (G disparity quads, K consecutive colsum
//             columns).  colsum(c, d) = sum over the w window rows of
//             |L(c) - R(c-d)|, kept in registers as u16x2 words
//             A = (4q, 4q+1), B = (4q+2, 4q+3).  One VABSDIFF4 of the spread
//             L byte (L, 0, L, 0) against a spread R pair (R(x), 0, R(x-1), 0)
//             gives two disparities directly in u16x2 lanes; each row step
//             adds the entering row and subtracts the leaving one in a single
//             IADD3 per word.  With PAIRS, the R pairs come ready-made from a
//             pair ring (each staged R row reversed into u16 lanes once per
//             CTA, see pair_at).  All byte alignments are
//             compile-time (K % 4 == 0, strip origin % 16 == 0, WIN fixed), so
//             every shift/permute has an immediate selector.  The row's
//             colsums go to shared memory buffer (row & 1).
//   horizontal (NHW warps) warp = one 32-column segment x 32 quads (HQ = 2,
//             lane = quad) or x 16 quads x {A, B} (HQ = 1, lane = word).  The
//             window sum over w colsums slides along x in NPART u16x2 partial
//             sums that never overflow; at matchable pixels the 2*HQ costs
//             become keys cost << 10 | d, min'ed in-lane, __reduce_min_sync
//             across the warp, and one shared atomicMin per warp: strict '<',
//             ties to the smallest d.  Disparity quads beyond the last full
//             warp (one quad at D = 16k) are summed directly per matchable
//             pixel by the lanes of the segment's first warp.
//
// Hand-off: named barriers FULL[b] (vertical arrive, horizontal sync) and
// EMPTY[b] (horizontal arrive, vertical sync) on the double-buffered colsum
// rows, so row t's horizontal pass overlaps row t+1's vertical pass.  Only
// pixels whose matchable bit is set (K4g) are evaluated and written.
#include <cstdlib>
#include <type_traits>

#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int kMaxThreads = 512;  // 4 warps per SMSP: 128 registers
constexpr size_t kSmemMax = 226 * 1024;  // dynamic shared memory per CTA
constexpr int kSegW = 32;  // output columns per horizontal segment
#ifndef STK_SAD_HB
#define STK_SAD_HB 6
#endif
constexpr int HB = STK_SAD_HB;  // matchable pixels per horizontal batch
enum { BAR_FULL0 = 1, BAR_FULL1 = 2, BAR_EMPTY0 = 3, BAR_EMPTY1 = 4, BAR_H = 5, BAR_V = 6 };

struct WP {
    int h, D, Q, QP, NG, NCH, CW, SW, CSW, TH;
    int NVW, NHW, QMAIN, NSEG;
    int RS, LP, RP, oL, oRw;  // ring slots, slot bytes, L offset, R word base offset
    int nthreads;             // 32 * (1 + NVW + NHW)
};

__device__ __forceinline__ uint32_t lo16(uint32_t v) { return v & 0xffffu; }
__device__ __forceinline__ uint32_t hi16(uint32_t v) { return v >> 16; }

// (byte p, 0, byte p-1, 0) of a run of words (p compile-time after unrolling).
template <int N>
__device__ __forceinline__ uint32_t r_pair(const uint32_t (&w)[N], int p) {
    const int i = p >> 2, s = p & 3;
    if (s) return __byte_perm(w[i], 0u, (uint32_t)s | 0x40u | (uint32_t)(s - 1) << 8 | 0x4000u);
    // byte p = byte 0 of w[i], byte p-1 = byte 3 of w[i-1]
    return __byte_perm(w[i - 1], w[i], 0x0304u) & 0x00ff00ffu;
}

// Vertical update of the G x K colsum units of one thread for one row pair.
// INIT: add the new row only.  Lw: L words of the row(s); Un/Uo: the rows'
// pair-ring words, pointer at word c - 1 of the thread (see pair_at).
template <int WIN, int G, int K>
struct VGeom {
    static constexpr int h = WIN / 2;
    static constexpr int rL = ((-h) % 4 + 4) % 4;     // byte residue of the L column base
    static constexpr int rR = ((1 - h) % 4 + 4) % 4;  // byte residue of the R window base
    static constexpr int NWL = (rL + K - 1) / 4 + 1;
    static constexpr int NWR = (G - 1) + (rR + K - 1) / 4 + 2;      // raw R words (no pair ring)
    static constexpr int PMIN = rR + 1, PMAX = rR + K + 4 * G - 2;  // pair positions p used
    static constexpr int JMIN = (PMIN - 1) / 2, JMAX = PMAX / 2;    // pair-ring words w[j] = U[c - j]
    static constexpr int NJ = JMAX - JMIN + 1;
};

// (R(P), 0, R(P-1), 0) for the thread's run position p (P = 4 rw0 + p): the
// pair ring stores R reversed as u16 (U[k] = R(Pmax - k)), so the pair is the
// u32 at U[k], k = Pmax - P = kb - p with kb odd: k even (one word) for odd p,
// a funnel of two words for even p.  w[j - JMIN] = U32[c - j], c = (kb - 1) / 2.
template <int JMIN, int NJ>
__device__ __forceinline__ uint32_t pair_at(const uint32_t (&w)[NJ], int p) {
    if (p & 1) return w[(p - 1) / 2 - JMIN];
    // U32[c - p/2] holds (U[k - 1], U[k]), U32[c - p/2 + 1] holds (U[k + 1], U[k + 2])
    return __byte_perm(w[p / 2 - JMIN], w[p / 2 - 1 - JMIN], 0x5432);
}

// PAIRS: Un / Uo point at the pair-ring words (word c - 1 of the thread, see
// pair_at); otherwise at the rows' raw R words (pairs built here, r_pair).
template <int WIN, int G, int K, bool INIT, bool PAIRS>
__device__ __forceinline__ void v_rows(const uint32_t* __restrict__ Ln, const uint32_t* __restrict__ Un,
                                       const uint32_t* __restrict__ Lo, const uint32_t* __restrict__ Uo,
                                       uint32_t (&A)[G][K], uint32_t (&B)[G][K]) {
    using V = VGeom<WIN, G, K>;
    constexpr int rL = V::rL, rR = V::rR, NWL = V::NWL, JMIN = V::JMIN;
    constexpr int NU = PAIRS ? V::NJ : V::NWR;
    uint32_t ln[NWL], lo[NWL], un[NU], uo[NU];
#pragma unroll
    for (int i = 0; i < NWL; ++i) ln[i] = Ln[i];
    // pair ring: Un points at U32[c - 1], w[j - JMIN] = U32[c - j] = Un[1 - j]
#pragma unroll
    for (int j = 0; j < NU; ++j) un[j] = PAIRS ? Un[1 - (j + JMIN)] : Un[j];
    if (!INIT) {
#pragma unroll
        for (int i = 0; i < NWL; ++i) lo[i] = Lo[i];
#pragma unroll
        for (int j = 0; j < NU; ++j) uo[j] = PAIRS ? Uo[1 - (j + JMIN)] : Uo[j];
    }
    auto pair = [&](const uint32_t (&w)[NU], int p) {
        if constexpr (PAIRS) return pair_at<JMIN, NU>(w, p);
        else return r_pair<NU>(w, p);
    };
    // Spread words: the L byte as (L, 0, L, 0) and R byte pairs as
    // (R(x), 0, R(x-1), 0), so one VABSDIFF4 yields two disparities already
    // in u16x2 lanes (no per-result unpacking).  R(c - 4q - m) sits at byte
    // o + 3 - m of the run, o = rR + k - 4j + 4(G-1); word A (d = 4q, 4q+1)
    // takes the pair at p = o + 3, word B (d = 4q+2, 4q+3) the pair at
    // p = o + 1.  The pairs come ready-made from the pair ring (built once per
    // row for the whole CTA instead of once per thread).
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int lb = rL + k;
        const uint32_t lsel = (uint32_t)(lb & 3) * 0x0101u | 0x4040u;  // bytes 1, 3 <- zero
        const uint32_t spn = __byte_perm(ln[lb >> 2], 0u, lsel);
        uint32_t spo = 0;
        if (!INIT) spo = __byte_perm(lo[lb >> 2], 0u, lsel);
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int o = rR + k - 4 * j + 4 * (G - 1);
            const uint32_t an = __vabsdiffu4(spn, pair(un, o + 3));
            const uint32_t bn = __vabsdiffu4(spn, pair(un, o + 1));
            if (INIT) {
                A[j][k] += an;
                B[j][k] += bn;
            } else {
                const uint32_t ao = __vabsdiffu4(spo, pair(uo, o + 3));
                const uint32_t bo = __vabsdiffu4(spo, pair(uo, o + 1));
                A[j][k] = A[j][k] + an - ao;
                B[j][k] = B[j][k] + bn - bo;
            }
        }
    }
}

// Window sum over colsum columns [a, a+WIN) from the chunk-local prefixes:
//   P[a+WIN-1] + sum_{c = a/K}^{(a+WIN-1)/K - 1} P[cK+K-1] - (a % K ? P[a-1] : 0).
// The 2 + NT column offsets of each segment position are precomputed (table
// `ent`, byte offsets within a quad row); absent terms point at the zeroed
// column ZC, so the sum is branch-free.  NW u16x2 words (NW == 1: word y if
// sel_y, else x); lo/hi are the two lanes' exact 32-bit sums.
template <int WIN, int K>
struct WinTab {
    static constexpr int NT = (WIN - 1 + K - 1) / K;  // most chunk totals a window spans
    static constexpr int NE = (2 + NT + 3) / 4 * 4;   // entry words (uint4 multiple)
};

template <int WIN, int K, int NW, bool MIXED = false>
__device__ __forceinline__ void window_sum(const char* __restrict__ cq, const uint32_t* __restrict__ ent,
                                           bool sel_y, uint32_t (&lo)[NW], uint32_t (&hi)[NW]) {
    constexpr int NT = WinTab<WIN, K>::NT, NE = WinTab<WIN, K>::NE;
    uint32_t o[NE];
#pragma unroll
    for (int i = 0; i < NE; i += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(ent + i);
        o[i] = v.x, o[i + 1] = v.y, o[i + 2] = v.z, o[i + 3] = v.w;
    }
    uint2 t[2 + NT];
#pragma unroll
    for (int i = 0; i < 2 + NT; ++i) t[i] = *reinterpret_cast<const uint2*>(cq + o[i]);
    // per word: X = sum(terms) - S in 32 bits (lanes mixed), Y = the exact sum
    // of the high lanes, low lanes = X - (Y << 16) (the true low sum is in
    // [0, 2^32), so the modular result is exact)
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const bool y = NW == 2 ? w == 1 : sel_y;
        uint32_t X = 0, Y = 0;
#pragma unroll
        for (int i = 0; i < 2 + NT; ++i) {
            if (i == 1) continue;  // the subtracted term
            const uint32_t x = y ? t[i].y : t[i].x;
            X += x;
            Y += hi16(x);
        }
        const uint32_t xs = y ? t[1].y : t[1].x;
        X -= xs;
        Y -= hi16(xs);
        lo[w] = MIXED ? X : X - (Y << 16);  // MIXED: the caller folds Y << 16 into its key
        hi[w] = Y;
    }
}

template <int WIN, int G, int K, int HQ, int NQB, bool PAIRS>
__global__ void __launch_bounds__(kMaxThreads, 1) k_sad_ws(Frame f, WP p) {
    constexpr int h = WIN / 2;
    static_assert(K * WIN * 255 <= 65535, "chunk prefix must fit a u16 lane");
    extern __shared__ __align__(128) uint8_t smem[];
    // layout: cs[2][QP][CSW] uint2 | ring RS x (LP + RP) | full[RS] | best[2][SW] | tab
    uint2* cs = reinterpret_cast<uint2*>(smem);
    uint8_t* ring = smem + (size_t)2 * p.QP * p.CSW * sizeof(uint2);
    uint64_t* fullb = reinterpret_cast<uint64_t*>(ring + (size_t)p.RS * (p.LP + p.RP));
    uint32_t* best = reinterpret_cast<uint32_t*>(fullb + p.RS);
    constexpr int NE = WinTab<WIN, K>::NE;
    uint32_t* tab = best + 2 * p.SW;  // [SW][NE] byte offsets (16-byte aligned)
    // pair ring: PR rows of R reversed as u16 (see pair_at), RP / 2 words each
    constexpr int PR = WIN + 4;
    uint32_t* pring = tab + (size_t)p.SW * NE;

    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int x0 = blockIdx.x * p.SW;
    const int yb0 = h + blockIdx.y * p.TH;
    const int yb1 = min(yb0 + p.TH, f.H - h);
    if (yb0 >= yb1) return;
    const int T = yb1 - yb0;           // output rows of this band
    const int NRR = T + WIN - 1;       // raw rows
    const int ry0 = yb0 - h;
    const int NVH = 32 * (p.NVW + p.NHW);

    for (int i = tid; i < 2 * p.SW; i += blockDim.x) best[i] = 0xffffffffu;
    // colsum column cc lives at slot cc + cc / K (one skew slot per chunk: the
    // vertical warps' 8-byte stores are bank-conflict free); slot ZC is never
    // written by them and holds the zero term
    const int ZC = p.NCH * (K + 1);
    for (int i = tid; i < 2 * p.QP; i += blockDim.x) cs[(size_t)i * p.CSW + ZC] = make_uint2(0u, 0u);
    if (tid == 0) {
        for (int s = 0; s < p.RS; ++s) {
            mbar_init(&fullb[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();

    // ---- row staging (issued by vertical thread 0): image columns
    // [xsL, xsL + LP) of L and [xsRa, xsRa + RP) of R, clamped to the plane.
    const int xsL = x0 - h - p.oL;
    const int xsR = x0 - h - 4 * p.QP + 1;
    const int xsRa = xsR - (((xsR % 16) + 16) % 16);  // 16-aligned start
    const int l0 = max(xsL, 0), l1 = min(xsL + p.LP, f.P);
    const int r0 = max(xsRa, 0), r1 = min(xsRa + p.RP, f.P);
    const uint32_t bl = l1 > l0 ? (uint32_t)(l1 - l0) : 0u;
    const uint32_t br = r1 > r0 ? (uint32_t)(r1 - r0) : 0u;
    auto issue_row = [&](int i) {
        const int s = i % p.RS;
        uint8_t* slot = ring + (size_t)s * (p.LP + p.RP);
        const size_t row = (size_t)(ry0 + i) * f.P;
        mbar_expect_tx(&fullb[s], bl + br);
        if (bl) bulk_g2s(slot + (l0 - xsL), f.grayL + row + l0, bl, &fullb[s]);
        if (br) bulk_g2s(slot + p.LP + (r0 - xsRa), f.grayR + row + r0, br, &fullb[s]);
    };

    if (wp < p.NVW) {
        // ------------------------------------------------------- vertical --
        const int tv = tid;
        if (tv == 0)
            for (int i = 0; i < min(p.RS, NRR); ++i) issue_row(i);
        int issued = min(p.RS, NRR);
        const int ch = tv % p.NCH, g = tv / p.NCH;
        const bool gok = g < p.NG;
        const bool act = gok;
        constexpr int rL = ((-h) % 4 + 4) % 4;
        // L: column cc = ch*K + k sits at slot byte cc + oL; word base (ch*K + oL - rL)/4
        const int lw0 = act ? (ch * K + p.oL - rL) >> 2 : 0;
        // R: window (cc, q) starts at slot byte cc - 4q + oRw*4 + rR
        const int rw0 = act ? (ch * K) / 4 - g * G - (G - 1) + p.oRw : 0;
        uint32_t A[G][K], B[G][K];
#pragma unroll
        for (int j = 0; j < G; ++j)
#pragma unroll
            for (int k = 0; k < K; ++k) A[j][k] = B[j][k] = 0u;
        uint2* csq = cs + (size_t)(g * G) * p.CSW + ch * (K + 1);
        const size_t bufstride = (size_t)p.QP * p.CSW;
        // Pair ring: row i's R bytes reversed into u16 lanes, U[k] = R(RP - 1 - k),
        // so every (R(x), 0, R(x-1), 0) pair the vertical pass needs is one
        // u32 (or a funnel of two): built once per row for the CTA, not once
        // per thread.  Item m = 8 u16 from two aligned raw words.
        const int RPW = p.RP / 2;  // u32 words per pair-ring row
        // spread(raw slot, its phase, pair slot)
        auto spread = [&](int rsl, uint32_t ph, int psl) {
            mbar_wait(&fullb[rsl], ph);
            const uint8_t* R = ring + (size_t)rsl * (p.LP + p.RP) + p.LP;
            uint32_t* U = pring + (size_t)psl * RPW;
            for (int m = tv; m < p.RP / 8; m += 32 * p.NVW) {
                const int k0 = 8 * m;
                const uint32_t wb = *reinterpret_cast<const uint32_t*>(R + p.RP - 4 - k0);
                const uint32_t wa = *reinterpret_cast<const uint32_t*>(R + p.RP - 8 - k0);
                *reinterpret_cast<uint4*>(U + k0 / 2) =
                    make_uint4(__byte_perm(wb, 0u, 0x4243), __byte_perm(wb, 0u, 0x4041),
                               __byte_perm(wa, 0u, 0x4243), __byte_perm(wa, 0u, 0x4041));
            }
        };
        // the thread's pair-ring word c - 1, c = (RP - 2) / 2 - 2 rw0 (see pair_at)
        const uint32_t* const ubase = pring + (RPW - 2 - 2 * rw0);
        // prologue: pair rows 0 .. PR-1 (rows are then built three steps ahead)
        if constexpr (PAIRS) {
            for (int i = 0; i < min(PR, NRR); ++i) spread(i % p.RS, (uint32_t)((i / p.RS) & 1), i);
            named_sync(BAR_V, 32 * p.NVW);
        }
        // pair slots of the entering / leaving rows and of the row built next
        // (PR + 2 = WIN + 6 > RS: its raw slot and phase tracked separately)
        int pn = WIN - 1, po = PR - 1, psp = (WIN + 4) % PR;
        int rsp = (WIN + 4) % p.RS;
        uint32_t php = (uint32_t)(((WIN + 4) / p.RS) & 1);
        int rs_n = WIN % p.RS, ph_n = (WIN / p.RS) & 1, rs_o = 0;
        for (int t = 0; t < T; ++t) {
            if (t == 0) {
                for (int i = 0; i < WIN; ++i) {
                    const int s = i % p.RS;
                    mbar_wait(&fullb[s], (uint32_t)((i / p.RS) & 1));
                    const uint32_t* Ls = reinterpret_cast<const uint32_t*>(ring + (size_t)s * (p.LP + p.RP));
                    const uint32_t* Rs = PAIRS ? ubase + (size_t)i * RPW
                                               : reinterpret_cast<const uint32_t*>(ring + (size_t)s * (p.LP + p.RP) + p.LP) + rw0;
                    if (act) v_rows<WIN, G, K, true, PAIRS>(Ls + lw0, Rs, nullptr, nullptr, A, B);
                }
            } else {
                // slot / phase of the entering row t+WIN-1 and the leaving row t-1
                const int sn = rs_n, so = rs_o;
                mbar_wait(&fullb[sn], (uint32_t)ph_n);
                if (++rs_n == p.RS) rs_n = 0, ph_n ^= 1;
                if (++rs_o == p.RS) rs_o = 0;
                const uint8_t* bn = ring + (size_t)sn * (p.LP + p.RP);
                const uint8_t* bo = ring + (size_t)so * (p.LP + p.RP);
                if (++pn == PR) pn = 0;
                if (++po == PR) po = 0;
                const uint32_t* Rn = PAIRS ? ubase + (size_t)pn * RPW : reinterpret_cast<const uint32_t*>(bn + p.LP) + rw0;
                const uint32_t* Ro = PAIRS ? ubase + (size_t)po * RPW : reinterpret_cast<const uint32_t*>(bo + p.LP) + rw0;
                if (act)
                    v_rows<WIN, G, K, false, PAIRS>(reinterpret_cast<const uint32_t*>(bn) + lw0, Rn,
                                                    reinterpret_cast<const uint32_t*>(bo) + lw0, Ro, A, B);
            }
            const int b = t & 1;
            if (t >= 2) {
                named_sync(BAR_EMPTY0 + b, NVH);
                // every vertical thread has finished reading rows <= t-1: their
                // slots take rows up to t-1+RS (async-proxy write after generic reads)
                if (tv == 0) {
                    fence_proxy_async();
                    for (; issued < min(t - 1 + p.RS + 1, NRR); ++issued) issue_row(issued);
                }
                // pair row t+WIN+2 (used from step t+3, after two more EMPTY
                // barriers) into the slot of row t-2, last read at step t-1
                if (PAIRS && t + WIN + 2 < NRR) spread(rsp, php, psp);
                if (++psp == PR) psp = 0;
                if (++rsp == p.RS) rsp = 0, php ^= 1u;
            }
            if (act) {
                uint2* dst = csq + b * bufstride;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    // chunk-local inclusive prefix of the colsums (K * w * 255 < 2^16)
                    uint32_t pa = 0, pb = 0;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        pa += A[j][k];
                        pb += B[j][k];
                        dst[(size_t)j * p.CSW + k] = make_uint2(pa, pb);
                    }
                }
            }
            named_arrive(BAR_FULL0 + b, NVH);
        }
        return;
    }

    // ------------------------------------------------------------ horizontal --
    // cs holds, per quad and colsum column cc, the inclusive prefix of the
    // colsums over cc's K-column chunk.  The window [a, a+w) of the pixel at
    // strip position x (a = x) is
    //   P[a+w-1] + sum_{c = a/K}^{(a+w-1)/K - 1} P[cK+K-1] - (a % K ? P[a-1] : 0),
    // every term a u16x2 word below 2^16 per lane; the sum is formed per lane
    // in 32 bits.  Only matchable pixels are visited.  Work split: horizontal
    // warp hw owns the 4-column groups g of the strip with g % NHW == hw (row
    // clusters of boundary pixels spread over all warps); its 32 positions
    // form one 32-bit mask per row.
    const int hw = wp - p.NVW;
    const int htid = tid - 32 * p.NVW;
    const int NW32 = p.SW / 32;                 // mask words per strip row
    // warp hw owns the 4-column groups gi = NHW*k + hw, k = 0..7 (SW = 32*NHW);
    // bit r of its mask is column 4*(NHW*(r>>2) + hw) + (r&3)
    auto pos_of = [&](int r) { return 4 * (p.NHW * (r >> 2) + hw) + (r & 3); };
    // the window-term table and the best keys are indexed by (warp, mask bit):
    // entry hwb + r is strip position pos_of(r), so a matchable pixel's table
    // address comes straight from its bit index
    const int hwb = 32 * hw;
    // warp mask of row y: lane k < 8 fetches group NHW*k + hw (word gi>>3,
    // nibble gi&7) and the warp OR-reduces the groups
    const uint32_t* mcol = f.mbits + (x0 >> 5);
    const int mgi = p.NHW * (lane & 7) + hw;
    const int mj = mgi >> 3;
    const int mshift = 4 * (mgi & 7);
    const bool mload = lane < 8 && x0 + 32 * mj < f.W;
    auto load_mask = [&](int y) {
        const uint32_t wd = mload ? __ldg(mcol + (size_t)y * f.bits_words + mj) : 0u;
        return __reduce_or_sync(0xffffffffu, ((wd >> mshift) & 0xfu) << (4 * (lane & 7)));
    };
    // lane -> quad of block qb: qb*32 + lane (HQ = 2) or qb*16 + lane%16, word lane/16 (HQ = 1)
    constexpr int QPB = HQ == 2 ? 32 : 16;  // quads per block
    const int region = HQ == 2 ? 0 : (lane >> 4);
    const int qlane = HQ == 2 ? lane : (lane & 15);
    // fast path: every main disparity <= D and every pixel of the strip has
    // x - h >= D (no left-edge truncation)
    const bool fast = (4 * p.QMAIN - 1 <= p.D) && (x0 - h >= p.D);
    const size_t bufstride = (size_t)p.QP * p.CSW;
    {
        constexpr int NT = WinTab<WIN, K>::NT;
        for (int a = htid; a < p.SW; a += 32 * p.NHW) {
            const int e = a + WIN - 1, ca = a / K, ce = e / K;
            const int g4 = a >> 2;  // a = pos_of(r) of warp g4 % NHW, r = 4 (g4 / NHW) + a % 4
            uint32_t* en = tab + (32 * (g4 % p.NHW) + 4 * (g4 / p.NHW) + (a & 3)) * NE;
            auto slot = [&](int cc) { return (uint32_t)(cc + cc / K) * 8u; };
            en[0] = slot(e);
            en[1] = a % K ? slot(a - 1) : (uint32_t)ZC * 8u;
#pragma unroll
            for (int t2 = 0; t2 < NT; ++t2) en[2 + t2] = ca + t2 < ce ? slot((ca + t2) * K + K - 1) : (uint32_t)ZC * 8u;
#pragma unroll
            for (int t2 = 2 + NT; t2 < NE; ++t2) en[t2] = 0u;
        }
        named_sync(BAR_H, 32 * p.NHW);
    }
    // per-lane quad-row bases of both colsum buffers, hoisted out of the row
    // loop (keeps WP fields out of the pixel loop: no constant reloads there)
    const char* qrow0[NQB];
    const char* qrow1[NQB];
    bool qokv[NQB];
#pragma unroll
    for (int qb = 0; qb < (NQB == 1 ? 1 : 0); ++qb) {
        const int q = qb * QPB + qlane;
        qokv[qb] = q < p.QMAIN;
        qrow0[qb] = reinterpret_cast<const char*>(cs + (size_t)(qokv[qb] ? q : 0) * p.CSW);
        qrow1[qb] = qrow0[qb] + bufstride * sizeof(uint2);
    }
    uint32_t* const best0 = best;
    uint32_t* const best1 = best + p.SW;
    const int Dm = p.D;
    uint32_t m = load_mask(yb0);
    uint32_t mprev = 0;
    for (int t = 0; t < T; ++t) {
        const int b = t & 1, y = yb0 + t;
        const uint32_t mnext = t + 1 < T ? load_mask(y + 1) : 0u;
        named_sync(BAR_FULL0 + b, NVH);
        // results of row t-1 are complete: write and reset them
        if ((mprev >> lane) & 1u) {
            const int x = pos_of(lane);
            const uint32_t* bp = NQB == 1 ? (b ? best0 : best1) : best + (b ^ 1) * p.SW;
            f.sparse[(size_t)(y - 1) * f.W + x0 + x] = (int16_t)(bp[hwb + lane] & 1023u);
        }
        if (m) {
            const uint2* cb = cs + b * bufstride;
            uint32_t* bp = NQB == 1 ? (b ? best1 : best0) : best + b * p.SW;
            auto pixels = [&](auto fast_tag) {
                constexpr bool FAST = decltype(fast_tag)::value;
                // in-lane min key of the main quads at mask bit r
                auto keyof = [&](int r) {
                    const int Dl = NQB == 1 ? Dm : p.D;
                    const int lim = FAST ? Dl : min(Dl, x0 + pos_of(r) - h);
                    uint32_t key = 0xffffffffu;
#pragma unroll
                    for (int qb = 0; qb < NQB; ++qb) {
                        const int q = qb * QPB + qlane;
                        // NQB == 1: the hoisted lane bases (0.4915 -> 0.481 ms at
                        // config C); NQB == 2 recomputes them (hoisting both
                        // blocks' bases costs registers: 5.9 -> 8.1 ms at config E)
                        bool qok;
                        const char* cq;
                        if constexpr (NQB == 1) {
                            qok = qokv[qb];
                            cq = b ? qrow1[qb] : qrow0[qb];
                        } else {
                            qok = q < p.QMAIN;
                            cq = reinterpret_cast<const char*>(cb + (size_t)(qok ? q : 0) * p.CSW);
                        }
                        const uint32_t dbase = 4 * q + 2 * region;
                        uint32_t lo[HQ], hi[HQ];
                        window_sum<WIN, K, HQ, true>(cq, tab + (hwb + r) * NE, region != 0, lo, hi);
#pragma unroll
                        for (int w = 0; w < HQ; ++w) {
                            // word w: d = dbase + 2w (lo lane), dbase + 2w + 1 (hi lane);
                            // lo[w] = X = low sum + (hi sum << 16) mod 2^32, so the low
                            // lane's key (X - (Y << 16)) * 1024 + d0 is X * 1024 + d0 -
                            // Y * 2^26 (mod 2^32): two multiply-adds
                            const uint32_t d0 = dbase + 2 * w;
                            uint32_t k0 = hi[w] * (uint32_t)(-(1 << 26)) + (lo[w] * 1024u + d0),
                                     k1 = hi[w] * 1024u + d0 + 1;
                            if (!FAST) {
                                if ((int)d0 > lim) k0 = 0xffffffffu;
                                if ((int)d0 + 1 > lim) k1 = 0xffffffffu;
                            }
                            const uint32_t kk = min(k0, k1);
                            key = qok ? min(key, kk) : key;
                        }
                    }
                    return key;
                };
                // four (then two) matchable pixels per iteration: independent
                // load -> sum -> min chains overlap on dense rows
                uint32_t mm = m;
                auto batch = [&](auto n_tag) {
                    constexpr int NB = decltype(n_tag)::value;
                    int xs[NB];  // mask bits
#pragma unroll
                    for (int i = 0; i < NB; ++i) {
                        xs[i] = __ffs(mm) - 1;
                        mm &= mm - 1;
                    }
                    uint32_t ks[NB];
#pragma unroll
                    for (int i = 0; i < NB; ++i) ks[i] = keyof(xs[i]);
#pragma unroll
                    for (int i = 0; i < NB; ++i) ks[i] = __reduce_min_sync(0xffffffffu, ks[i]);
                    if (lane == 0) {
#pragma unroll
                        for (int i = 0; i < NB; ++i) bp[hwb + xs[i]] = ks[i];
                    }
                };
                while (__popc(mm) >= HB) batch(std::integral_constant<int, HB>{});
                if (HB > 4 && __popc(mm) >= 4) batch(std::integral_constant<int, 4>{});
                for (; mm;) {
                    const int x1 = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const int x2 = mm ? __ffs(mm) - 1 : x1;
                    mm &= mm - 1;
                    uint32_t k1 = keyof(x1), k2 = keyof(x2);
                    k1 = __reduce_min_sync(0xffffffffu, k1);
                    k2 = __reduce_min_sync(0xffffffffu, k2);
                    // this warp owns the pixel and covers every main quad
                    if (lane == 0) {
                        bp[hwb + x1] = k1;
                        bp[hwb + x2] = k2;
                    }
                }
            };
            if (fast) pixels(std::true_type{});
            else pixels(std::false_type{});
            // quads beyond the main blocks: lane r takes the pixel of mask bit r
            __syncwarp();
            if (p.QMAIN < p.Q && ((m >> lane) & 1u)) {
                const int x = pos_of(lane);
                const int lim = min(p.D, x0 + x - h);
                uint32_t key = 0xffffffffu;
                for (int qx = p.QMAIN; qx < p.Q; ++qx) {
                    uint32_t lo[2], hi[2];
                    window_sum<WIN, K, 2>(reinterpret_cast<const char*>(cb + (size_t)qx * p.CSW),
                                          tab + (hwb + lane) * NE, false, lo, hi);
                    const uint32_t c[4] = {lo[0], hi[0], lo[1], hi[1]};
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int d = 4 * qx + jj;
                        if (d <= lim) key = min(key, c[jj] * 1024u + (uint32_t)d);
                    }
                }
                bp[hwb + lane] = min(bp[hwb + lane], key);
            }
        }
        if (t + 2 < T) named_arrive(BAR_EMPTY0 + b, NVH);
        mprev = m;
        m = mnext;
    }
    // last row
    named_sync(BAR_H, 32 * p.NHW);
    if ((mprev >> lane) & 1u) {
        const int x = pos_of(lane), y = yb1 - 1, b = (T - 1) & 1;
        f.sparse[(size_t)y * f.W + x0 + x] = (int16_t)(best[b * p.SW + hwb + lane] & 1023u);
    }
}

template <int WIN, int G, int K, int HQ, int NQB, bool PAIRS>
void run_ws(const Frame& f, const WP& p, size_t sm, int bands, cudaStream_t st) {
    auto kern = k_sad_ws<WIN, G, K, HQ, NQB, PAIRS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const dim3 grid((f.W + p.SW - 1) / p.SW, bands);
    kern<<<grid, p.nthreads, sm, st>>>(f, p);
}

// per-window thread shape: K colsum columns (K * w * 255 < 2^16 for the chunk
// prefix) x G disparity quads per vertical thread
template <int WIN>
struct Shape {
    static constexpr int K = WIN <= 21 ? 12 : 8;
    static constexpr int G = WIN <= 21 ? 3 : 5;  // 33 / 65 quads at D = 128 / 256
};

template <int WIN, bool PAIRS>
void run_win_p(const Frame& f, const WP& p, int HQ, int NQB, size_t sm, int bands, cudaStream_t st) {
    constexpr int G = Shape<WIN>::G, K = Shape<WIN>::K;
    if (HQ == 2) {
        if (NQB == 1) run_ws<WIN, G, K, 2, 1, PAIRS>(f, p, sm, bands, st);
        else run_ws<WIN, G, K, 2, 2, PAIRS>(f, p, sm, bands, st);
    } else {
        if (NQB == 1) run_ws<WIN, G, K, 1, 1, PAIRS>(f, p, sm, bands, st);
        else run_ws<WIN, G, K, 1, 2, PAIRS>(f, p, sm, bands, st);
    }
}

template <int WIN>
void run_win(const Frame& f, const WP& p, int HQ, int NQB, bool pairs, size_t sm, int bands, cudaStream_t st) {
    if (pairs) run_win_p<WIN, true>(f, p, HQ, NQB, sm, bands, st);
    else run_win_p<WIN, false>(f, p, HQ, NQB, sm, bands, st);
}

}  // namespace

bool launch_sad_ws(const Frame& f, cudaStream_t st, bool dry) {
    const int w = f.window, h = f.hw, D = f.D;
    if (!(w == 9 || w == 15 || w == 21 || w == 31)) return false;
    if (f.W > 65535 || D > 1023 || f.H - 2 * h <= 0) return false;
    const int G = w <= 21 ? Shape<21>::G : Shape<31>::G;
    const int K = w <= 21 ? Shape<21>::K : Shape<31>::K;
    WP p{};
    p.h = h;
    p.D = D;
    p.Q = (D + 1 + 3) / 4;
    p.QP = (p.Q + G - 1) / G * G;
    p.NG = p.QP / G;
    // horizontal lanes: quads (HQ = 2) when there are >= 32 of them, else words
    const int HQ = p.Q >= 32 ? 2 : 1;
    const int per_block = HQ == 2 ? 32 : 16;
    p.QMAIN = std::max(1, p.Q / per_block) * per_block;
    if (p.QMAIN > p.Q || p.Q - p.QMAIN > 2) p.QMAIN = p.Q;  // partial block, no direct quads
    const int NQB = (p.QMAIN + per_block - 1) / per_block;
    if (NQB > 2) return false;
    // strip width: as wide as shared memory allows (fewer halo columns)
    const int sms = f.sms > 0 ? f.sms : 148;
    size_t sm = 0;
    for (int SW : {256, 192, 128, 96, 64}) {
        p.SW = SW;
        p.CW = SW + w - 1;
        p.NCH = (p.CW + K - 1) / K;
        // quad row stride: odd (the horizontal lanes = quads hit distinct 8-byte
        // bank pairs), residue chosen to minimise the vertical warps' 8-byte
        // store conflicts (a half-warp = 16 lanes per shared-memory wavefront)
        {
            const int base = p.NCH * (K + 1) + 1;  // skewed columns + the zero slot
            int bestc = base | 1, bestcost = 1 << 30;
            for (int c = base | 1; c < base + 16; c += 2) {
                int cost = 0;
                for (int t0 = 0; t0 < p.NG * p.NCH; t0 += 16) {
                    int cnt[16] = {0};
                    int mx = 0;
                    for (int l = t0; l < std::min(t0 + 16, p.NG * p.NCH); ++l) {
                        const int ch = l % p.NCH, g = l / p.NCH;
                        const int sl = ((g * G) * c + ch * (K + 1)) & 15;
                        mx = std::max(mx, ++cnt[sl]);
                    }
                    cost += mx;
                }
                if (cost < bestcost) bestcost = cost, bestc = c;
            }
            p.CSW = bestc;
        }
        p.NSEG = SW / kSegW;
        p.NHW = p.NSEG;
        p.NVW = (p.NG * p.NCH + 31) / 32;
        p.nthreads = 32 * (p.NVW + p.NHW);
        p.RS = w + 1 + 4;
        p.oL = ((-h) % 16 + 16) % 16;
        p.LP = (p.NCH * K + p.oL + 8 + 15) & ~15;
        // R slot: image column X sits at X - xsRa; window (cc, q) byte
        // cc - 4q - 3 + (x0 - h - xsRa) = cc - 4q + 4*QP - 4 + oR, oR = (xsR mod 16)
        const int oR = ((1 - h - 4 * p.QP) % 16 + 16) % 16;
        const int rR = ((1 - h) % 4 + 4) % 4;
        p.oRw = (4 * p.QP - 4 + oR - rR) / 4;
        p.RP = (p.NCH * K + 4 * p.QP + oR + 16 + 15) & ~15;
        const int NE = w <= 21 ? (w == 21 ? WinTab<21, 12>::NE : WinTab<15, 12>::NE) : WinTab<31, 8>::NE;
        sm = (size_t)2 * p.QP * p.CSW * 8 + (size_t)p.RS * (p.LP + p.RP) + p.RS * 8 +
             2 * SW * 4 + (size_t)SW * NE * 4;
        if (sm <= kSmemMax && p.nthreads <= kMaxThreads) break;
        sm = 0;
    }
    if (!sm) return false;
    // the pair ring only where it fits beside the strip width chosen without it
    // (a narrower strip costs more halo columns than the ring saves: config E
    // 5.9 -> 9.2 ms) and where the vertical role is the long one -- many
    // disparity quads per row (4K, 33 quads: 0.481 -> 0.477 ms; 1080p, 18
    // quads: 0.117 -> 0.122 ms, the per-row build is not amortised)
    const size_t ring_bytes = (size_t)(w + 4) * p.RP * 2;
    const bool pairs = sm + ring_bytes <= kSmemMax && p.QP >= 24;
    if (pairs) sm += ring_bytes;
    const int strips = (f.W + p.SW - 1) / p.SW;
    const int rows = f.H - 2 * h;
    // one wave of one CTA per SM when possible; bands of >= 32 rows.
    // STK_SAD_SMS (experiment knob) caps the SMs the kernel takes so other
    // frames' kernels can run beside it.
    static const int sms_cap = [] {
        const char* e = getenv("STK_SAD_SMS");
        return e ? atoi(e) : 0;
    }();
    int bands = std::max(1, (sms_cap > 0 ? std::min(sms, sms_cap) : sms) / strips);
    bands = std::min(bands, std::max(1, rows / 32));
    p.TH = (rows + bands - 1) / bands;
    bands = (rows + p.TH - 1) / p.TH;
    if (dry) return true;
    switch (w) {
        case 9: run_win<9>(f, p, HQ, NQB, pairs, sm, bands, st); break;
        case 15: run_win<15>(f, p, HQ, NQB, pairs, sm, bands, st); break;
        case 21: run_win<21>(f, p, HQ, NQB, pairs, sm, bands, st); break;
        default: run_win<31>(f, p, HQ, NQB, pairs, sm, bands, st); break;
    }
    return true;
}

}  // namespace stk
