// K5b sad_strip -- boundary-pixel SAD matching with column-sum reuse.
//
// Integer sums are associative, so sharing partial sums between neighbouring
// pixels yields exactly the cost the reference's per-pixel loop computes
// (stereo.cpp:12-28) and therefore the same winner (stereo.cpp:90-97).
//
// A CTA owns a strip of 128 output columns x a band of TH output rows.
//   staging    every row the band needs (both views) arrives through 1-D bulk
//              TMA copies (cp.async.bulk -> UBLKCP), one per row and view,
//              into shared memory; 16-byte aligned column runs.
//   vertical   thread (column chunk of MAXC consecutive columns, disparity
//              quad q) keeps colsum[c][4q..4q+3] = sum over the window rows
//              of |L(c) - R(c-d)| in registers as two u16x2 words.  One
//              VABSDIFF4 of the replicated L byte against the 4 bytes
//              R(c-4q-3 .. c-4q) gives all four |L-R|; each row step subtracts
//              the leaving row and adds the entering one (subtract first: no
//              u16 borrow).  Byte extraction uses compile-time selectors on
//              runtime-realigned words.
//   horizontal warp = 16 disparity quads x {low, high} pair of one 32-column
//              chunk; the window sum over w colsums slides along x in NPART
//              u16x2 partial sums small enough never to overflow, widened to
//              u32 only at matchable pixels; the 32 steps are fully unrolled
//              so every shared load has an immediate offset.
//   argmin     key = cost << 10 | d, __reduce_min_sync per warp, one shared
//              atomicMin per warp: strict '<', ties to the smallest d.
// Only pixels whose matchable bit is set (K4g) are evaluated and written.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int SW = 128;   // output columns per strip
constexpr int SNT = 512;  // threads per CTA

struct SG {
    int h, w, D, Q, NCH, NWP, NSEG, SEGW, CW, PART, TH, offL, offR2, LP, RP, NR, CS, R1;
};


// |L(c) - R(c-d)| for the 4 disparities of quad q at the MAXC columns of this
// thread's chunk, for one staged row.  lw / rw point at the 4-byte aligned
// words containing the first needed byte; sL / sR are the byte misalignments.
template <int MAXC>
__device__ __forceinline__ void row_absdiff(const uint32_t* lw, const uint32_t* rw, int sL, int sR,
                                            uint32_t (&v)[MAXC]) {
    uint32_t la[MAXC / 4], ra[MAXC / 4 + 1];
    {
        uint32_t prev = lw[0];
#pragma unroll
        for (int j = 0; j < MAXC / 4; ++j) {
            const uint32_t nxt = lw[j + 1];
            la[j] = __funnelshift_r(prev, nxt, sL * 8);
            prev = nxt;
        }
    }
    {
        uint32_t prev = rw[0];
#pragma unroll
        for (int j = 0; j < MAXC / 4 + 1; ++j) {
            const uint32_t nxt = rw[j + 1];
            ra[j] = __funnelshift_r(prev, nxt, sR * 8);
            prev = nxt;
        }
    }
#pragma unroll
    for (int k = 0; k < MAXC; ++k) {
        const uint32_t rep = __byte_perm(la[k >> 2], 0u, (k & 3) * 0x1111);
        const uint32_t rv = (k & 3) == 0 ? ra[k >> 2]
                                         : __funnelshift_r(ra[k >> 2], ra[(k >> 2) + 1], (k & 3) * 8);
        v[k] = __vabsdiffu4(rep, rv);
    }
}

// WIN > 0: the window size is a compile-time constant (the configured sizes
// 9/15/21/31): the horizontal pass then keeps the 32+WIN-1 column sums of a
// chunk in registers and slides with compile-time indices (one IADD3 per part
// per step, no shared loads inside the slide).  WIN == 0: runtime window.
template <int MAXC, int NPART, int WIN>
__global__ void __launch_bounds__(SNT, (MAXC <= 12) ? 2 : 1) k_sad_strip(Frame f, SG g) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t best[SW];
    uint8_t* Lr = smem;
    uint8_t* Rr = Lr + (size_t)g.NR * g.LP;
    uint32_t* cs = reinterpret_cast<uint32_t*>(Rr + (size_t)g.NR * g.RP);
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int x0 = blockIdx.x * SW;
    const int yb0 = g.h + blockIdx.y * g.TH;
    const int yb1 = min(yb0 + g.TH, f.H - g.h);
    if (yb0 >= yb1) return;
    const int ry0 = yb0 - g.h;
    const int nrows = (yb1 - yb0) + 2 * g.h;
    for (int i = tid; i < SW; i += SNT) best[i] = 0xffffffffu;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    // ---- staging: rows ry0 .. ry0+nrows-1 of both views (clamped to the plane)
    if (wp == 0) {
        const int xsL = x0 - g.h - g.offL, xsR = x0 - g.h - g.offR2;
        const int l0 = max(xsL, 0), l1 = min(xsL + g.LP, f.P);
        const int r0 = max(xsR, 0), r1 = min(xsR + g.RP, f.P);
        const uint32_t bl = l1 > l0 ? (uint32_t)(l1 - l0) : 0u;
        const uint32_t br = r1 > r0 ? (uint32_t)(r1 - r0) : 0u;
        if (lane == 0) mbar_expect_tx(&bar, (uint32_t)nrows * (bl + br));
        __syncwarp();
        for (int r = lane; r < nrows; r += 32) {
            const size_t row = (size_t)(ry0 + r) * f.P;
            if (bl) bulk_g2s(Lr + (size_t)r * g.LP + (l0 - xsL), f.grayL + row + l0, bl, &bar);
            if (br) bulk_g2s(Rr + (size_t)r * g.RP + (r0 - xsR), f.grayR + row + r0, br, &bar);
        }
    }
    mbar_wait(&bar, 0);

    // ---- vertical role: chunk ch (columns c0 .. c0+MAXC-1), quad q
    const int q = tid % g.Q, ch = tid / g.Q;
    const bool vact = ch < g.NCH;
    const int c0 = ch * MAXC;
    const int lbase = g.offL + c0, rbase = c0 - 4 * q - 3 + g.offR2;
    const int sL = lbase & 3, sR = rbase & 3;
    const uint8_t* Lp = Lr + (lbase & ~3);
    const uint8_t* Rp = Rr + (rbase & ~3);
    uint32_t* csA = cs + (size_t)q * g.CS + c0;          // pairs (4q, 4q+1)
    uint32_t* csB = cs + g.R1 + (size_t)q * g.CS + c0;   // pairs (4q+2, 4q+3)
    uint32_t A[MAXC], B[MAXC];
#pragma unroll
    for (int k = 0; k < MAXC; ++k) A[k] = B[k] = 0u;

    // ---- horizontal role: chunk-of-32 segment, 16 quads x {A, B}
    const int seg = wp / g.NWP;
    const bool hact = seg < g.NSEG;
    const int region = lane >> 4;
    const int qq = (wp % g.NWP) * 16 + (lane & 15);
    const bool qvalid = qq < g.Q;
    const uint32_t* colp = cs + region * g.R1 + (size_t)min(qq, g.Q - 1) * g.CS;
    const int dlo = 4 * qq + 2 * region;  // disparity of the low half (high half = dlo + 1)

    const uint32_t* mbase = f.mbits + (x0 >> 5);
    for (int y = yb0; y < yb1; ++y) {
        if (vact) {
            uint32_t v[MAXC];
            if (y == yb0) {
                for (int r = 0; r < g.w; ++r) {
                    row_absdiff<MAXC>(reinterpret_cast<const uint32_t*>(Lp + (size_t)r * g.LP),
                                      reinterpret_cast<const uint32_t*>(Rp + (size_t)r * g.RP), sL, sR, v);
#pragma unroll
                    for (int k = 0; k < MAXC; ++k) {
                        A[k] += __byte_perm(v[k], 0u, 0x4243);
                        B[k] += __byte_perm(v[k], 0u, 0x4041);
                    }
                }
            } else {
                // colsum + new - old in one IADD3 per packed word: every u16
                // lane's result lies in [0, w*255], so the exact 32-bit
                // arithmetic never carries or borrows across lanes.
                const int ro = y - yb0 - 1, rn = y - yb0 + 2 * g.h;
                uint32_t vn[MAXC];
                row_absdiff<MAXC>(reinterpret_cast<const uint32_t*>(Lp + (size_t)ro * g.LP),
                                  reinterpret_cast<const uint32_t*>(Rp + (size_t)ro * g.RP), sL, sR, v);
                row_absdiff<MAXC>(reinterpret_cast<const uint32_t*>(Lp + (size_t)rn * g.LP),
                                  reinterpret_cast<const uint32_t*>(Rp + (size_t)rn * g.RP), sL, sR, vn);
#pragma unroll
                for (int k = 0; k < MAXC; ++k) {
                    A[k] = A[k] + __byte_perm(vn[k], 0u, 0x4243) - __byte_perm(v[k], 0u, 0x4243);
                    B[k] = B[k] + __byte_perm(vn[k], 0u, 0x4041) - __byte_perm(v[k], 0u, 0x4041);
                }
            }
#pragma unroll
            for (int k = 0; k < MAXC; ++k) {
                csA[k] = A[k];
                csB[k] = B[k];
            }
        }
        const uint32_t* mrow = mbase + (size_t)y * f.bits_words;
        const bool any = (__ldg(mrow) | __ldg(mrow + 1) | __ldg(mrow + 2) | __ldg(mrow + 3)) != 0u;
        __syncthreads();
        if (!any) continue;
        if (hact) {
            const int dl_base = -g.h;  // d valid iff d <= min(D, x - h)
            for (int cb = 0; cb < g.SEGW; cb += 32) {
                const int xi0 = seg * g.SEGW + cb;
                const uint32_t m = __ldg(mrow + (xi0 >> 5));
                if constexpr (WIN > 0) {
                    // ring of the WIN+1 most recent column sums, indexed with
                    // compile-time positions (the 32 steps are unrolled)
                    constexpr int PW = (WIN + NPART - 1) / NPART;  // columns per part
                    constexpr int RW = WIN + 1;
                    uint32_t ring[RW];
                    const uint32_t* cp = colp + xi0;
#pragma unroll
                    for (int k = 0; k < WIN; ++k) ring[k] = cp[k];
                    uint32_t S[NPART];
#pragma unroll
                    for (int j = 0; j < NPART; ++j) {
                        S[j] = 0;
#pragma unroll
                        for (int k = j * PW; k < (j + 1) * PW && k < WIN; ++k) S[j] += ring[k];
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (i > 0) {
                            ring[(i + WIN - 1) % RW] = cp[i + WIN - 1];
#pragma unroll
                            for (int j = 0; j < NPART; ++j) {
                                const int ks = j * PW;
                                const int ke = ((j + 1) * PW < WIN ? (j + 1) * PW : WIN) - 1;
                                S[j] = S[j] + ring[(i + ke) % RW] - ring[(i - 1 + ks) % RW];
                            }
                        }
                        if ((m >> i) & 1u) {
                            const int x = x0 + xi0 + i;
                            const int dl = min(g.D, x + dl_base);
                            uint32_t c0v = 0, c1v = 0;
#pragma unroll
                            for (int j = 0; j < NPART; ++j) {
                                c0v += S[j] & 0xffffu;
                                c1v += S[j] >> 16;
                            }
                            uint32_t key = 0xffffffffu;
                            if (qvalid && dlo <= dl) key = (c0v << 10) | (uint32_t)dlo;
                            if (qvalid && dlo + 1 <= dl) key = min(key, (c1v << 10) | (uint32_t)(dlo + 1));
                            key = __reduce_min_sync(0xffffffffu, key);
                            if (lane == 0) atomicMin(&best[xi0 + i], key);
                        }
                    }
                    continue;
                }
                // part j covers window offsets [j*PART, min((j+1)*PART, w))
                uint32_t S[NPART];
                const uint32_t* po[NPART];
                const uint32_t* pn[NPART];
#pragma unroll
                for (int j = 0; j < NPART; ++j) {
                    const int ks = j * g.PART, ke = min(ks + g.PART, g.w);
                    uint32_t s = 0;
                    for (int k = ks; k < ke; ++k) s += colp[xi0 + k];
                    S[j] = s;
                    po[j] = colp + xi0 + ks;      // leaving column at step i: po[j][i-1]
                    pn[j] = colp + xi0 + ke;      // entering column at step i: pn[j][i-1]
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i > 0) {
#pragma unroll
                        for (int j = 0; j < NPART; ++j) S[j] = S[j] - po[j][i - 1] + pn[j][i - 1];
                    }
                    if ((m >> i) & 1u) {
                        const int x = x0 + xi0 + i;
                        const int dl = min(g.D, x + dl_base);
                        uint32_t c0v = 0, c1v = 0;
#pragma unroll
                        for (int j = 0; j < NPART; ++j) {
                            c0v += S[j] & 0xffffu;
                            c1v += S[j] >> 16;
                        }
                        uint32_t key = 0xffffffffu;
                        if (qvalid && dlo <= dl) key = (c0v << 10) | (uint32_t)dlo;
                        if (qvalid && dlo + 1 <= dl) key = min(key, (c1v << 10) | (uint32_t)(dlo + 1));
                        key = __reduce_min_sync(0xffffffffu, key);
                        if (lane == 0) atomicMin(&best[xi0 + i], key);
                    }
                }
            }
        }
        __syncthreads();
        if (tid < SW) {
            const uint32_t mw = __ldg(mrow + (tid >> 5));
            if ((mw >> (tid & 31)) & 1u) {
                f.sparse[(size_t)y * f.W + x0 + tid] = (int16_t)(best[tid] & 1023u);
                best[tid] = 0xffffffffu;
            }
        }
    }
}

template <int MAXC, int NPART, int WIN>
void run(const Frame& f, const SG& g, size_t sm, cudaStream_t st) {
    cudaFuncSetAttribute(k_sad_strip<MAXC, NPART, WIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    const dim3 grid((f.W + SW - 1) / SW, (f.H - 2 * g.h + g.TH - 1) / g.TH);
    k_sad_strip<MAXC, NPART, WIN><<<grid, SNT, sm, st>>>(f, g);
}

template <int MAXC>
void run_np(const Frame& f, const SG& g, int npart, size_t sm, cudaStream_t st) {
    switch (g.w) {  // compile-time windows (npart follows from w, see launch_sad_strip)
        case 9: run<MAXC, 1, 9>(f, g, sm, st); return;
        case 15: run<MAXC, 1, 15>(f, g, sm, st); return;
        case 21: run<MAXC, 2, 21>(f, g, sm, st); return;
        case 31: run<MAXC, 4, 31>(f, g, sm, st); return;
        default: break;
    }
    if (npart == 1) run<MAXC, 1, 0>(f, g, sm, st);
    else if (npart == 2) run<MAXC, 2, 0>(f, g, sm, st);
    else run<MAXC, 4, 0>(f, g, sm, st);
}

}  // namespace

bool launch_sad_strip(const Frame& f, cudaStream_t st, bool dry) {
    SG g{};
    g.h = f.hw;
    g.w = f.window;
    g.D = f.D;
    if (g.w > 31 || g.D > 1023 || f.W > 65535) return false;  // key packs d in 10 bits
    g.Q = (g.D + 1 + 3) / 4;
    g.CW = SW + 2 * g.h;
    static const int kMaxc[] = {4, 8, 12, 16, 24};
    int maxc = 0;
    for (int m : kMaxc) {
        const int nch = (g.CW + m - 1) / m;
        if (nch * g.Q <= SNT) {
            maxc = m;
            g.NCH = nch;
            break;
        }
    }
    if (!maxc) return false;
    // horizontal: NWP warps (16 quads each) per 32-column chunk segment
    g.NWP = (g.Q + 15) / 16;
    const int warps = SNT / 32;
    if (g.NWP > warps) return false;
    int nseg = 1;
    while (nseg * 2 * g.NWP <= warps && nseg * 2 <= SW / 32) nseg *= 2;
    g.NSEG = nseg;
    g.SEGW = SW / nseg;
    // u16x2 partial sums: part * w * 255 <= 65535
    const int need = (g.w * 255 * g.w + 65534) / 65535;  // parts needed
    int npart = need <= 1 ? 1 : (need <= 2 ? 2 : 4);
    g.PART = (g.w + npart - 1) / npart;
    if ((long)g.PART * g.w * 255 > 65535) return false;
    g.TH = 64;
    g.offL = (-g.h) & 15;
    const int dq = 4 * g.Q - 1;
    g.offR2 = dq + ((-(g.h + dq)) & 15);
    const int csrows = g.NCH * maxc;
    g.CS = csrows | 1;
    while ((g.CS & 31) != 1) g.CS += 2;  // CS = 1 mod 32: conflict-free quads
    g.R1 = g.Q * g.CS;
    g.R1 += ((16 - (g.R1 & 31)) + 32) & 31;  // region B starts 16 banks apart
    g.LP = (g.offL + csrows + 8 + 15) & ~15;
    g.RP = (g.offR2 + csrows + 8 + 15) & ~15;
    g.NR = g.TH + 2 * g.h;
    const size_t sm = (size_t)g.NR * (g.LP + g.RP) + (size_t)(g.R1 + g.Q * g.CS) * 4;
    if (sm > 220 * 1024) return false;
    if (dry) return true;
    switch (maxc) {
        case 4: run_np<4>(f, g, npart, sm, st); break;
        case 8: run_np<8>(f, g, npart, sm, st); break;
        case 12: run_np<12>(f, g, npart, sm, st); break;
        case 16: run_np<16>(f, g, npart, sm, st); break;
        default: run_np<24>(f, g, npart, sm, st); break;
    }
    return true;
}

}  // namespace stk
