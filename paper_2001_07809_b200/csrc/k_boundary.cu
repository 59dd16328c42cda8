// K3 boundary_morph -- detect -> fill -> remove in ONE pass over a TMA-staged
// halo tile (reference: boundary.cpp:11-85, pipeline.cpp:87-91).
//
// A CTA owns a 128x32 output tile.  The 8-bit lightness tile plus a 3-pixel
// halo (8 columns on each side to keep the TMA box 16-byte aligned) arrives by
// one cp.async.bulk.tensor; labels are recomputed on chip from gray via the
// K-Means LUT (so the u16 LabelMap never touches HBM in lean mode).
//
// Edge rules are coded explicitly, not taken from TMA's zero fill:
//   * detect ignores out-of-image neighbours: replicating the nearest in-image
//     row/column into the halo is equivalent, because a clamped neighbour is
//     either the pixel itself or one of its real neighbours;
//   * fill/remove only change interior pixels (1..W-2, 1..H-2) and both are
//     no-ops when W < 3 or H < 3.
// The same kernel serves the per-stage entries (detect on u16 labels, fill
// only, remove only) through the MorphMode template parameter.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int TW = 128, TH = 32, HALO = 3;
// TMA box: columns x0-16 .. x0+144 (the box's first column must sit on a
// 16-byte boundary -- measured on B200: 8-bit boxes starting elsewhere fault),
// rows y0-3 .. y0+35.
constexpr int BW = TW + 32;
constexpr int BH = TH + 2 * HALO;
constexpr int XOFF = 16;           // smem column of x0
constexpr int kThreads = 256;

template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_morph(const __grid_constant__ CUtensorMap tmap, Frame f, uint8_t* __restrict__ out_a,
            uint8_t* __restrict__ out_b) {
    using T = typename std::conditional<MODE == MORPH_DETECT16, uint16_t, uint8_t>::type;
    __shared__ __align__(128) T in[BH][BW];
    __shared__ uint8_t raw[BH][BW];
    __shared__ uint8_t fil[BH][BW];
    __shared__ __align__(8) uint64_t bar;
    __shared__ unsigned long long red[kThreads / 32];

    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    const int W = f.W, H = f.H;
    const int tid = threadIdx.x;
    if (tid == 0) {
        tma_prefetch_desc(&tmap);
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bar, (uint32_t)sizeof(in));
        tma_load_2d(&in[0][0], &tmap, &bar, x0 - XOFF, y0 - HALO);
    }
    mbar_wait(&bar, 0);

    // --- replicate the nearest in-image column/row into out-of-image halo cells
    const bool edge = x0 - XOFF < 0 || y0 - HALO < 0 || x0 + TW + XOFF > W || y0 + TH + HALO > H;
    if (edge) {
        const int cmin = XOFF - x0, cmax = XOFF + (W - 1 - x0);  // in-image smem cols
        for (int i = tid; i < BH * BW; i += kThreads) {
            const int r = i / BW, cc = i % BW;
            if (cc < cmin) in[r][cc] = in[r][cmin];
            else if (cc > cmax) in[r][cc] = in[r][cmax];
        }
        __syncthreads();
        const int rmin = HALO - y0, rmax = HALO + (H - 1 - y0);
        for (int i = tid; i < BH * BW; i += kThreads) {
            const int r = i / BW, cc = i % BW;
            if (r < rmin) in[r][cc] = in[rmin][cc];
            else if (r > rmax) in[r][cc] = in[rmax][cc];
        }
    }
    if (MODE == MORPH_FUSED) {
        // labels on chip: cluster index of each gray value (segmentation.cpp:146-155)
        __syncthreads();
        const uint8_t* lut = f.sc->lut;
        for (int i = tid; i < BH * BW; i += kThreads) {
            uint8_t* p = reinterpret_cast<uint8_t*>(&in[0][0]) + i;
            *p = lut[*p];
        }
    }
    __syncthreads();

    // --- detect (boundary.cpp:11-39) for rows y0-2..y0+TH+1, cols x0-2..x0+TW+1
    if (MODE == MORPH_FUSED || MODE == MORPH_DETECT16) {
        constexpr int R0 = HALO - 2, C0 = XOFF - 2, NR = TH + 4, NC = TW + 4;
        for (int i = tid; i < NR * NC; i += kThreads) {
            const int r = R0 + i / NC, cc = C0 + i % NC;
            const T c = in[r][cc];
            const bool b = in[r - 1][cc - 1] != c || in[r - 1][cc] != c || in[r - 1][cc + 1] != c ||
                           in[r][cc - 1] != c || in[r][cc + 1] != c || in[r + 1][cc - 1] != c ||
                           in[r + 1][cc] != c || in[r + 1][cc + 1] != c;
            raw[r][cc] = b;
        }
    } else {
        for (int i = tid; i < BH * BW; i += kThreads)
            (&raw[0][0])[i] = reinterpret_cast<const uint8_t*>(&in[0][0])[i] ? 1 : 0;
    }
    __syncthreads();

    // --- fill (boundary.cpp:41-63) for rows y0-1..y0+TH, cols x0-1..x0+TW
    if (MODE == MORPH_FUSED || MODE == MORPH_FILL) {
        constexpr int R0 = HALO - 1, C0 = XOFF - 1, NR = TH + 2, NC = TW + 2;
        for (int i = tid; i < NR * NC; i += kThreads) {
            const int r = R0 + i / NC, cc = C0 + i % NC;
            const int x = x0 + cc - XOFF, y = y0 + r - HALO;
            uint8_t v = raw[r][cc];
            if (!v && x >= 1 && x <= W - 2 && y >= 1 && y <= H - 2)
                v = raw[r - 1][cc - 1] & raw[r - 1][cc] & raw[r - 1][cc + 1] & raw[r][cc - 1] &
                    raw[r][cc + 1] & raw[r + 1][cc - 1] & raw[r + 1][cc] & raw[r + 1][cc + 1];
            fil[r][cc] = v;
        }
    } else {
        for (int i = tid; i < BH * BW; i += kThreads) (&fil[0][0])[i] = (&raw[0][0])[i];
    }
    __syncthreads();

    // --- remove (boundary.cpp:65-85) on the output tile, write + count
    unsigned long long n_raw = 0, n_out = 0;
    for (int i = tid; i < TH * (TW / 4); i += kThreads) {
        const int r = HALO + i / (TW / 4), cq = XOFF + (i % (TW / 4)) * 4;
        const int y = y0 + r - HALO, xb = x0 + cq - XOFF;
        if (y >= H || xb >= W) continue;
        uint32_t packed_out = 0, packed_raw = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = cq + j, x = xb + j;
            uint8_t v;
            if (MODE == MORPH_FUSED || MODE == MORPH_REMOVE) {
                v = fil[r][cc];
                if (v && x >= 1 && x <= W - 2 && y >= 1 && y <= H - 2 &&
                    (fil[r - 1][cc] & fil[r][cc - 1] & fil[r][cc + 1] & fil[r + 1][cc]))
                    v = 0;
            } else if (MODE == MORPH_FILL) {
                v = fil[r][cc];
            } else {
                v = raw[r][cc];
            }
            if (x < W) {
                packed_out |= (uint32_t)v << (8 * j);
                packed_raw |= (uint32_t)raw[r][cc] << (8 * j);
                n_out += v;
                n_raw += raw[r][cc];
            }
        }
        const size_t o = (size_t)y * f.P + xb;
        if (MODE == MORPH_FUSED) {
            *reinterpret_cast<uint32_t*>(out_b + o) = packed_out;  // refined (pitched, padded)
            if (out_a) *reinterpret_cast<uint32_t*>(out_a + o) = packed_raw;
        } else {
            *reinterpret_cast<uint32_t*>(out_a + o) = packed_out;
        }
    }
    if (MODE == MORPH_FUSED) {
        const unsigned long long t_raw = block_sum_u64<kThreads>(n_raw, red);
        const unsigned long long t_out = block_sum_u64<kThreads>(n_out, red);
        if (tid == 0) {
            if (t_raw) atomicAdd(&f.sc->raw_count, t_raw);
            if (t_out) atomicAdd(&f.sc->refined_count, t_out);
        }
    }
}

}  // namespace

void launch_morph(const Frame& f, int mode, const CUtensorMap* tmap, uint8_t* out_a,
                  uint8_t* out_b, cudaStream_t st) {
    if (f.N == 0) return;
    const dim3 grid((f.W + TW - 1) / TW, (f.H + TH - 1) / TH);
    switch (mode) {
        case MORPH_FUSED: k_morph<MORPH_FUSED><<<grid, kThreads, 0, st>>>(*tmap, f, out_a, out_b); break;
        case MORPH_DETECT16: k_morph<MORPH_DETECT16><<<grid, kThreads, 0, st>>>(*tmap, f, out_a, out_b); break;
        case MORPH_FILL: k_morph<MORPH_FILL><<<grid, kThreads, 0, st>>>(*tmap, f, out_a, out_b); break;
        default: k_morph<MORPH_REMOVE><<<grid, kThreads, 0, st>>>(*tmap, f, out_a, out_b); break;
    }
}

}  // namespace stk
