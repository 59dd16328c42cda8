// K8 blur_sep -- depth-range-masked Gaussian blur of the left view
// (reference: refocus.cpp:45-113, pipeline.cpp:141-146).
//
// A CTA owns a 64x16 output tile.  The RGB tile plus a kernel-half-width halo
// is staged in shared memory with the reference's replicate-border rule coded
// explicitly (clamped source coordinates, refocus.cpp:97-99).  The blur
// decision is fused: a pixel stays sharp iff its dense disparity is known and
// inside a focus range (refocus.cpp:45-73, as a per-disparity LUT), so the
// blur map never exists in HBM.  Tiles with no blurred pixel just copy.
//
//   default : separable FP32 (horizontal pass into shared memory, vertical
//             pass in registers) -- within 1 LSB of the reference's 2-D FP64
//             sum (tests bound it);
//   exact   : 2-D FP64 in the reference's i-outer / j-inner order with
//             __dmul_rn/__dadd_rn and lround -- bit-identical.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int BX = 64, BY = 16, kThreads = 256;

__device__ __forceinline__ bool sharp_px(const BlurParams& bp, const Frame& f, const int16_t* depth,
                                         int x, int y) {
    if (bp.blur_map) return bp.blur_map[(size_t)y * f.P + x] == 0;
    const int d = depth[(size_t)y * f.W + x];
    return d >= 0 && d < bp.lut_len && bp.sharp_lut[d];
}

template <bool EXACT>
__global__ void __launch_bounds__(kThreads) k_blur(Frame f, BlurParams bp,
                                                   const uint8_t* __restrict__ in,
                                                   uint8_t* __restrict__ out,
                                                   const int16_t* __restrict__ depth) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int h = bp.hw, W = f.W, H = f.H;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY;
    const int IW = BX + 2 * h, IH = BY + 2 * h;
    const int tid = threadIdx.x;
    // any pixel of this tile blurred?
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
        return;
    }
    uint8_t* tile = smem;  // IH x IW x 3
    for (int i = tid; i < IW * IH; i += kThreads) {
        const int r = i / IW, c = i % IW;
        const int sy = min(max(y0 - h + r, 0), H - 1), sx = min(max(x0 - h + c, 0), W - 1);
        const uint8_t* p = in + ((size_t)sy * W + sx) * 3;
        uint8_t* q = tile + (size_t)i * 3;
        q[0] = p[0];
        q[1] = p[1];
        q[2] = p[2];
    }
    const int K = 2 * h + 1;
    if (EXACT) {
        double* w2 = reinterpret_cast<double*>(smem + (((size_t)IW * IH * 3 + 15) & ~(size_t)15));
        for (int i = tid; i < K * K; i += kThreads) w2[i] = bp.g2[i];
        __syncthreads();
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
            for (int r = 0; r < K; ++r) {
                const uint8_t* row = tile + ((size_t)(oy + r) * IW + ox) * 3;
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
        return;
    }
    // separable FP32: horizontal pass for all IH rows into hs[IH][BX][3]
    float* g = reinterpret_cast<float*>(smem + (((size_t)IW * IH * 3 + 15) & ~(size_t)15));
    float* hs = g + ((K + 3) & ~3);
    for (int i = tid; i < K; i += kThreads) g[i] = bp.g1[i];
    __syncthreads();
    for (int i = tid; i < IH * BX; i += kThreads) {
        const int r = i / BX, ox = i % BX;
        const uint8_t* row = tile + ((size_t)r * IW + ox) * 3;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
        for (int c = 0; c < K; ++c) {
            const float wt = g[c];
            a0 = fmaf(wt, (float)row[c * 3], a0);
            a1 = fmaf(wt, (float)row[c * 3 + 1], a1);
            a2 = fmaf(wt, (float)row[c * 3 + 2], a2);
        }
        float* o = hs + ((size_t)r * BX + ox) * 3;
        o[0] = a0;
        o[1] = a1;
        o[2] = a2;
    }
    __syncthreads();
    for (int i = tid; i < BX * BY; i += kThreads) {
        const int ox = i % BX, oy = i / BX;
        const int x = x0 + ox, y = y0 + oy;
        if (x >= W || y >= H) continue;
        const size_t o = ((size_t)y * W + x) * 3;
        if (sharp_px(bp, f, depth, x, y)) {
            const uint8_t* t = tile + ((size_t)(oy + h) * IW + ox + h) * 3;
            out[o] = t[0];
            out[o + 1] = t[1];
            out[o + 2] = t[2];
            continue;
        }
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
        for (int r = 0; r < K; ++r) {
            const float wt = g[r];
            const float* s = hs + ((size_t)(oy + r) * BX + ox) * 3;
            a0 = fmaf(wt, s[0], a0);
            a1 = fmaf(wt, s[1], a1);
            a2 = fmaf(wt, s[2], a2);
        }
        out[o] = (uint8_t)min(max((int)floorf(a0 + 0.5f), 0), 255);
        out[o + 1] = (uint8_t)min(max((int)floorf(a1 + 0.5f), 0), 255);
        out[o + 2] = (uint8_t)min(max((int)floorf(a2 + 0.5f), 0), 255);
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

}  // namespace

size_t blur_smem_bytes(int hw, bool exact) {
    const int IW = BX + 2 * hw, IH = BY + 2 * hw, K = 2 * hw + 1;
    size_t b = (((size_t)IW * IH * 3) + 15) & ~(size_t)15;
    if (exact) return b + (size_t)K * K * sizeof(double);
    return b + (((size_t)K + 3) & ~(size_t)3) * sizeof(float) + (size_t)IH * BX * 3 * sizeof(float);
}

void launch_blur(const Frame& f, const BlurParams& bp, const uint8_t* in_rgb, uint8_t* out_rgb,
                 const int16_t* depth, cudaStream_t st) {
    if (f.N == 0) return;
    const dim3 grid((f.W + BX - 1) / BX, (f.H + BY - 1) / BY);
    const size_t sm = blur_smem_bytes(bp.hw, bp.exact != 0);
    if (bp.exact) {
        cudaFuncSetAttribute(k_blur<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_blur<true><<<grid, kThreads, sm, st>>>(f, bp, in_rgb, out_rgb, depth);
    } else {
        cudaFuncSetAttribute(k_blur<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_blur<false><<<grid, kThreads, sm, st>>>(f, bp, in_rgb, out_rgb, depth);
    }
}

void launch_blur_map(const Frame& f, const int16_t* depth, const uint8_t* sharp_lut, int lut_len,
                     uint8_t* out, cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 16);
    k_blur_map<<<(int)blocks, 256, 0, st>>>(f, depth, sharp_lut, lut_len, out);
}

}  // namespace stk
