// K8 blur_sep -- depth-range-masked Gaussian blur of the left view
// (reference: refocus.cpp:45-113, pipeline.cpp:141-146).
//
// A CTA owns a 64x32 output tile.  The RGB tile plus a kernel-half-width halo
// is staged in shared memory with the reference's replicate-border rule coded
// explicitly (clamped source coordinates, refocus.cpp:97-99).  The blur
// decision is fused: a pixel stays sharp iff its dense disparity is known and
// inside a focus range (refocus.cpp:45-73, as a per-disparity LUT), so the
// blur map never exists in HBM.  Tiles with no blurred pixel just copy.
//
//   default : separable FP32, register-blocked: a thread computes 4
//             horizontally adjacent outputs of one staged row (16+2h bytes
//             per channel converted once with the 2^23 magic-number trick),
//             then 4 vertically adjacent outputs of one column from float4
//             shared rows -- within 1 LSB of the reference's 2-D FP64 sum
//             (tests bound it);
//   exact   : 2-D FP64 in the reference's i-outer / j-inner order with
//             __dmul_rn/__dadd_rn and lround -- bit-identical.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int BX = 64, BY = 32, kThreads = 256;

__device__ __forceinline__ bool sharp_px(const BlurParams& bp, const Frame& f, const int16_t* depth,
                                         int x, int y) {
    if (bp.blur_map) return bp.blur_map[(size_t)y * f.P + x] == 0;
    const int d = depth[(size_t)y * f.W + x];
    return d >= 0 && d < bp.lut_len && bp.sharp_lut[d];
}

__device__ __forceinline__ float byte_f(uint32_t w, int k) {  // byte k of w as float, exact
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540 | k)) - 8388608.0f;
}

struct TileGeom {
    int h, IW, IH, rowb;  // staged tile: IH rows of IW pixels, rowb bytes per row (16-aligned)
};

__device__ __forceinline__ TileGeom tile_geom(int h) {
    TileGeom g;
    g.h = h;
    g.IW = BX + 2 * h;
    g.IH = BY + 2 * h;
    g.rowb = ((g.IW * 3 + 15) & ~15) + 16;
    return g;
}

// returns false when every pixel of the tile is sharp (and copies it)
__device__ __forceinline__ bool stage_tile(const Frame& f, const BlurParams& bp,
                                           const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                           const int16_t* __restrict__ depth, uint8_t* tile,
                                           const TileGeom& g, int x0, int y0) {
    const int W = f.W, H = f.H, tid = threadIdx.x;
    bool any = false;
    for (int i = tid; i < BX * BY; i += kThreads) {
        const int x = x0 + (i % BX), y = y0 + i / BX;
        if (x < W && y < H && !sharp_px(bp, f, depth, x, y)) any = true;
    }
    any = __syncthreads_or(any);
    if (!any) {
        for (int i = tid; i < BX * BY * 3; i += kThreads) {
            const int p = i / 3, c = i % 3;
            const int x = x0 + (p % BX), y = y0 + p / BX;
            if (x < W && y < H) out[((size_t)y * W + x) * 3 + c] = in[((size_t)y * W + x) * 3 + c];
        }
        return false;
    }
    for (int i = tid; i < g.IW * g.IH; i += kThreads) {
        const int r = i / g.IW, c = i % g.IW;
        const int sy = min(max(y0 - g.h + r, 0), H - 1), sx = min(max(x0 - g.h + c, 0), W - 1);
        const uint8_t* p = in + ((size_t)sy * W + sx) * 3;
        uint8_t* q = tile + (size_t)r * g.rowb + c * 3;
        q[0] = p[0];
        q[1] = p[1];
        q[2] = p[2];
    }
    __syncthreads();
    return true;
}

__global__ void __launch_bounds__(kThreads) k_blur_sep(Frame f, BlurParams bp,
                                                       const uint8_t* __restrict__ in,
                                                       uint8_t* __restrict__ out,
                                                       const int16_t* __restrict__ depth) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TileGeom g = tile_geom(bp.hw);
    const int h = g.h, K = 2 * h + 1, W = f.W, H = f.H, tid = threadIdx.x;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
    float* gw = reinterpret_cast<float*>(smem);                        // K weights
    float4* hs = reinterpret_cast<float4*>(smem + (((size_t)K * 4 + 15) & ~(size_t)15));  // IH x BX
    uint8_t* tile = reinterpret_cast<uint8_t*>(hs + (size_t)g.IH * BX);
    for (int i = tid; i < K; i += kThreads) gw[i] = bp.g1[i];
    if (!stage_tile(f, bp, in, out, depth, tile, g, x0, y0)) return;
    // horizontal: item = (staged row r, 4 consecutive outputs 4q..4q+3)
    for (int it = tid; it < g.IH * (BX / 4); it += kThreads) {
        const int r = it / (BX / 4), q4 = (it % (BX / 4)) * 4;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(tile + (size_t)r * g.rowb + q4 * 3);
        float a[4][3];
#pragma unroll
        for (int o = 0; o < 4; ++o) a[o][0] = a[o][1] = a[o][2] = 0.f;
        // pixels q4 .. q4+3+2h; pixel p channel c = byte 3p+c of the run
        const int np = 4 + 2 * h;
        uint32_t wcur = src[0];
        int wi = 0;
        for (int p = 0; p < np; ++p) {
            float v[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int b = 3 * p + c;
                if ((b >> 2) != wi) {
                    wi = b >> 2;
                    wcur = src[wi];
                }
                v[c] = byte_f(wcur, b & 3);
            }
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int k = p - o;
                if (k >= 0 && k < K) {
                    const float wt = gw[k];
                    a[o][0] = fmaf(wt, v[0], a[o][0]);
                    a[o][1] = fmaf(wt, v[1], a[o][1]);
                    a[o][2] = fmaf(wt, v[2], a[o][2]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) hs[(size_t)r * BX + q4 + o] = make_float4(a[o][0], a[o][1], a[o][2], 0.f);
    }
    __syncthreads();
    // vertical: item = (column x, 4 consecutive output rows)
    for (int it = tid; it < BX * (BY / 4); it += kThreads) {
        const int ox = it % BX, oy4 = (it / BX) * 4;
        const int x = x0 + ox;
        if (x >= W) continue;
        float a[4][3];
#pragma unroll
        for (int o = 0; o < 4; ++o) a[o][0] = a[o][1] = a[o][2] = 0.f;
        for (int r = 0; r < 4 + 2 * h; ++r) {
            const float4 v = hs[(size_t)(oy4 + r) * BX + ox];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int k = r - o;
                if (k >= 0 && k < K) {
                    const float wt = gw[k];
                    a[o][0] = fmaf(wt, v.x, a[o][0]);
                    a[o][1] = fmaf(wt, v.y, a[o][1]);
                    a[o][2] = fmaf(wt, v.z, a[o][2]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int y = y0 + oy4 + o;
            if (y >= H) break;
            uint8_t* dst = out + ((size_t)y * W + x) * 3;
            if (sharp_px(bp, f, depth, x, y)) {
                const uint8_t* t = tile + (size_t)(oy4 + o + h) * g.rowb + (ox + h) * 3;
                dst[0] = t[0];
                dst[1] = t[1];
                dst[2] = t[2];
            } else {
                dst[0] = (uint8_t)min(max((int)floorf(a[o][0] + 0.5f), 0), 255);
                dst[1] = (uint8_t)min(max((int)floorf(a[o][1] + 0.5f), 0), 255);
                dst[2] = (uint8_t)min(max((int)floorf(a[o][2] + 0.5f), 0), 255);
            }
        }
    }
}

// Same algorithm with the kernel size known at compile time: the 4-output
// horizontal / vertical loops unroll completely, weights live in registers and
// byte positions are constants (the common sizes of default_kernel_size).
template <int K>
__global__ void __launch_bounds__(kThreads) k_blur_sep_k(Frame f, BlurParams bp,
                                                         const uint8_t* __restrict__ in,
                                                         uint8_t* __restrict__ out,
                                                         const int16_t* __restrict__ depth) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int h = K / 2, NP = 4 + 2 * h, NWB = (3 * NP + 3) / 4;
    const TileGeom g = tile_geom(h);
    const int W = f.W, H = f.H, tid = threadIdx.x;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
    float4* hs = reinterpret_cast<float4*>(smem);  // IH x BX
    uint8_t* tile = reinterpret_cast<uint8_t*>(hs + (size_t)g.IH * BX);
    float wk[K];
#pragma unroll
    for (int i = 0; i < K; ++i) wk[i] = __ldg(bp.g1 + i);
    if (!stage_tile(f, bp, in, out, depth, tile, g, x0, y0)) return;
    for (int it = tid; it < g.IH * (BX / 4); it += kThreads) {
        const int r = it / (BX / 4), q4 = (it % (BX / 4)) * 4;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(tile + (size_t)r * g.rowb + q4 * 3);
        uint32_t wv[NWB];
#pragma unroll
        for (int i = 0; i < NWB; ++i) wv[i] = src[i];
        float a[4][3];
#pragma unroll
        for (int o = 0; o < 4; ++o) a[o][0] = a[o][1] = a[o][2] = 0.f;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float v[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) v[c] = byte_f(wv[(3 * p + c) >> 2], (3 * p + c) & 3);
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                if (p - o >= 0 && p - o < K) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) a[o][c] = fmaf(wk[p - o], v[c], a[o][c]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) hs[(size_t)r * BX + q4 + o] = make_float4(a[o][0], a[o][1], a[o][2], 0.f);
    }
    __syncthreads();
    for (int it = tid; it < BX * (BY / 4); it += kThreads) {
        const int ox = it % BX, oy4 = (it / BX) * 4;
        const int x = x0 + ox;
        if (x >= W) continue;
        float a[4][3];
#pragma unroll
        for (int o = 0; o < 4; ++o) a[o][0] = a[o][1] = a[o][2] = 0.f;
#pragma unroll
        for (int r = 0; r < NP; ++r) {
            const float4 v = hs[(size_t)(oy4 + r) * BX + ox];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                if (r - o >= 0 && r - o < K) {
                    a[o][0] = fmaf(wk[r - o], v.x, a[o][0]);
                    a[o][1] = fmaf(wk[r - o], v.y, a[o][1]);
                    a[o][2] = fmaf(wk[r - o], v.z, a[o][2]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int y = y0 + oy4 + o;
            if (y >= H) break;
            uint8_t* dst = out + ((size_t)y * W + x) * 3;
            if (sharp_px(bp, f, depth, x, y)) {
                const uint8_t* t = tile + (size_t)(oy4 + o + h) * g.rowb + (ox + h) * 3;
                dst[0] = t[0];
                dst[1] = t[1];
                dst[2] = t[2];
            } else {
                dst[0] = (uint8_t)min(max((int)floorf(a[o][0] + 0.5f), 0), 255);
                dst[1] = (uint8_t)min(max((int)floorf(a[o][1] + 0.5f), 0), 255);
                dst[2] = (uint8_t)min(max((int)floorf(a[o][2] + 0.5f), 0), 255);
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_blur_exact(Frame f, BlurParams bp,
                                                         const uint8_t* __restrict__ in,
                                                         uint8_t* __restrict__ out,
                                                         const int16_t* __restrict__ depth) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TileGeom g = tile_geom(bp.hw);
    const int K = 2 * g.h + 1, W = f.W, H = f.H, tid = threadIdx.x;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
    double* w2 = reinterpret_cast<double*>(smem);
    uint8_t* tile = smem + (size_t)K * K * sizeof(double);
    for (int i = tid; i < K * K; i += kThreads) w2[i] = bp.g2[i];
    if (!stage_tile(f, bp, in, out, depth, tile, g, x0, y0)) return;
    for (int i = tid; i < BX * BY; i += kThreads) {
        const int ox = i % BX, oy = i / BX;
        const int x = x0 + ox, y = y0 + oy;
        if (x >= W || y >= H) continue;
        const size_t o = ((size_t)y * W + x) * 3;
        if (sharp_px(bp, f, depth, x, y)) {
            out[o] = in[o];
            out[o + 1] = in[o + 1];
            out[o + 2] = in[o + 2];
            continue;
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int r = 0; r < K; ++r) {  // i outer, j inner (refocus.cpp:95-105)
            const uint8_t* row = tile + (size_t)(oy + r) * g.rowb + ox * 3;
            const double* wr = w2 + r * K;
            for (int c = 0; c < K; ++c) {
                const double wt = wr[c];
                a0 = __dadd_rn(a0, __dmul_rn(wt, (double)row[c * 3]));
                a1 = __dadd_rn(a1, __dmul_rn(wt, (double)row[c * 3 + 1]));
                a2 = __dadd_rn(a2, __dmul_rn(wt, (double)row[c * 3 + 2]));
            }
        }
        out[o] = (uint8_t)min(max(lround(a0), 0L), 255L);
        out[o + 1] = (uint8_t)min(max(lround(a1), 0L), 255L);
        out[o + 2] = (uint8_t)min(max(lround(a2), 0L), 255L);
    }
}

// explicit blur map (build_blur_map, refocus.cpp:45-73) for the stage entry
__global__ void k_blur_map(Frame f, const int16_t* __restrict__ depth, const uint8_t* __restrict__ lut,
                           int lut_len, uint8_t* __restrict__ out) {
    const long long n = f.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        const int d = depth[i];
        const bool sharp = d >= 0 && d < lut_len && lut[d];
        out[(size_t)y * f.P + x] = sharp ? 0 : 1;
    }
}

size_t tile_bytes(int hw) {
    const int IW = BX + 2 * hw, IH = BY + 2 * hw;
    return (size_t)IH * ((((size_t)IW * 3 + 15) & ~(size_t)15) + 16);
}

}  // namespace

size_t blur_smem_bytes(int hw, bool exact) {
    const int K = 2 * hw + 1, IH = BY + 2 * hw;
    if (exact) return (size_t)K * K * sizeof(double) + tile_bytes(hw);
    return (((size_t)K * 4 + 15) & ~(size_t)15) + (size_t)IH * BX * sizeof(float4) + tile_bytes(hw);
}

void launch_blur(const Frame& f, const BlurParams& bp, const uint8_t* in_rgb, uint8_t* out_rgb,
                 const int16_t* depth, cudaStream_t st) {
    if (f.N == 0) return;
    const dim3 grid((f.W + BX - 1) / BX, (f.H + BY - 1) / BY);
    const size_t sm = blur_smem_bytes(bp.hw, bp.exact != 0);
    if (bp.exact) {
        cudaFuncSetAttribute(k_blur_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_blur_exact<<<grid, kThreads, sm, st>>>(f, bp, in_rgb, out_rgb, depth);
    } else {
        const int K = 2 * bp.hw + 1;
        // templated sizes: no weight array in shared memory
        const size_t smk = (size_t)(BY + 2 * bp.hw) * BX * sizeof(float4) + tile_bytes(bp.hw);
#define STK_BLUR_K(KK)                                                                          \
    case KK:                                                                                    \
        cudaFuncSetAttribute(k_blur_sep_k<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                             (int)smk);                                                         \
        k_blur_sep_k<KK><<<grid, kThreads, smk, st>>>(f, bp, in_rgb, out_rgb, depth);           \
        return;
        switch (K) {
            STK_BLUR_K(3)
            STK_BLUR_K(5)
            STK_BLUR_K(7)
            STK_BLUR_K(9)
            STK_BLUR_K(11)
            STK_BLUR_K(13)
            STK_BLUR_K(17)
            STK_BLUR_K(25)
            STK_BLUR_K(49)
            default: break;
        }
#undef STK_BLUR_K
        cudaFuncSetAttribute(k_blur_sep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_blur_sep<<<grid, kThreads, sm, st>>>(f, bp, in_rgb, out_rgb, depth);
    }
}

void launch_blur_map(const Frame& f, const int16_t* depth, const uint8_t* sharp_lut, int lut_len,
                     uint8_t* out, cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 16);
    k_blur_map<<<(int)blocks, 256, 0, st>>>(f, depth, sharp_lut, lut_len, out);
}

}  // namespace stk
