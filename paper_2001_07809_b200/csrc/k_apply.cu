// Stage-entry mask plumbing around the SAD kernels (reference:
// boundary.cpp:180-195, stereo.cpp:79-85, evaluate.cpp:92-135).  The frame
// path builds its matchable bits from the run CCL (k_bnd.cu B8); the stage
// entries match_boundary_pixels / dense_sad_baseline start from a caller's
// byte mask instead:
//
//   apply        byte mask (+ optional anchors) -> window filter -> matchable
//                bit-mask, the raster-ordered matchable-pixel list (warp
//                ballots, single-pass decoupled look-back) and per-row-tile
//                list offsets, sparse = Unknown, sad_ops.
//   anchor_only  add_border_anchors alone.
#include "stk_device.cuh"

namespace stk {

namespace {

__global__ void __launch_bounds__(256) k_apply(Frame f, int anchors) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[8];
    __shared__ unsigned long long red[8], red2[8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* status = f.lb + LB_LIST * f.lb_stride;
    if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_LIST], 1u);
    __syncthreads();
    const int c = s_chunk;
    const int t0 = c * kTilesPerChunk + wid * kTilesPerWarp;
    const int m = f.hw, W = f.W, H = f.H;
    uint32_t balls[kTilesPerWarp][4];
    uint32_t wc = 0, kept = 0;
    unsigned long long ops = 0;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        const bool tv = t < f.n_tiles;
        const int y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = seg * kRowTile + j * 32 + lane;
            bool keep = false, anc = false;
            if (tv && x < W) {
                const size_t po = (size_t)y * f.P + x;
                const int g = y * W + x;
                if (f.mref[po]) {
                    keep = true;
                }
                anc = keep;
                if (anchors && (x == m || x == W - 1 - m) && y >= m && y <= H - 1 - m) anc = true;
                if (f.mprn) f.mprn[po] = keep;
                if (f.manc) f.manc[po] = anc;
                f.sparse[g] = -1;
            }
            kept += keep;
            const bool matchable = anc && y >= m && y < H - m && x >= m && x < W - m;
            balls[k][j] = __ballot_sync(0xffffffffu, matchable);
            wc += __popc(balls[k][j]);
            if (matchable) ops += (unsigned long long)(min(f.D, x - m) + 1);
            if (tv && lane == 0) f.mbits[(size_t)y * f.bits_words + seg * 4 + j] = balls[k][j];
        }
    }
    if (lane == 0) wcount[wid] = wc;
    unsigned long long kk = kept, oo = ops;
    for (int o = 16; o > 0; o >>= 1) {
        kk += __shfl_xor_sync(0xffffffffu, kk, o);
        oo += __shfl_xor_sync(0xffffffffu, oo, o);
    }
    if (lane == 0) {
        red[wid] = kk;
        red2[wid] = oo;
    }
    __syncthreads();
    if (wid == 0) {
        const uint32_t agg = __reduce_add_sync(0xffffffffu, lane < 8 ? wcount[lane] : 0u);
        const uint32_t excl = lb_exclusive_warp(status, c, agg);
        if (lane == 0) {
            s_excl = excl;
            unsigned long long ka = 0, oa = 0;
            for (int i = 0; i < 8; ++i) {
                ka += red[i];
                oa += red2[i];
            }
            if (ka) atomicAdd(&f.sc->pruned_count, ka);
            if (oa) atomicAdd(&f.sc->sad_ops, oa * (unsigned long long)(f.window * f.window));
            if (c == f.n_chunks - 1) {
                f.sc->n_list = excl + agg;
                f.sc->matched = excl + agg;
                f.tile_off[f.n_tiles] = excl + agg;
            }
        }
    }
    __syncthreads();
    uint32_t pos = s_excl;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        if (t >= f.n_tiles) break;
        const int y = t / f.TX, seg = t % f.TX;
        if (lane == 0) f.tile_off[t] = pos;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (balls[k][j] >> lane & 1u) {
                const int x = seg * kRowTile + j * 32 + lane;
                f.list[pos + __popc(balls[k][j] & lanemask)] = ((uint32_t)y << 16) | (uint32_t)x;
            }
            pos += __popc(balls[k][j]);
        }
    }
}

// add_border_anchors alone (boundary.cpp:180-195)
__global__ void k_anchor_only(Frame f, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                              int m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < f.N;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        const size_t o = (size_t)y * f.P + x;
        uint8_t v = in[o];
        if ((x == m || x == f.W - 1 - m) && y >= m && y <= f.H - 1 - m) v = 1;
        out[o] = v;
    }
}

}  // namespace

void launch_apply(const Frame& f, bool anchors, cudaStream_t st) {
    if (f.N == 0) return;
    k_apply<<<f.n_chunks, 256, 0, st>>>(f, anchors ? 1 : 0);
}

void launch_anchor_only(const Frame& f, const uint8_t* in, uint8_t* out, int margin,
                        cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, f.sms * 16);
    k_anchor_only<<<(int)blocks, 256, 0, st>>>(f, in, out, margin);
}

}  // namespace stk
