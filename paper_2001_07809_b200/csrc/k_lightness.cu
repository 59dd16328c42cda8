// K1 lstar_hist -- RGB -> CIE L* (8-bit) for both views in one launch, with the
// left view's 256-bin histogram fused in (shared-memory privatised atomics).
//
// Reference: lightness.cpp:25-53 (per pixel, FP64), segmentation.cpp:11-44
// (histogram).  Bit-exactness without device transcendentals:
//   * Y = 0.2126*lin[R] + 0.7152*lin[G] + 0.0722*lin[B] is evaluated with
//     __dmul_rn/__dadd_rn in the reference's left-to-right order (no DFMA
//     contraction), lin[] computed by the host libm (lightness.cpp:29-32).
//   * The reference's 8-bit L* is non-decreasing in Y, so gray(Y) is the
//     number of host thresholds thr[v] (v = 1..255, smallest Y with L* >= v)
//     that are <= Y: an 8-step binary search in shared memory replaces
//     cbrt/lround.  Verified over all 2^24 RGB triples (tests).
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int kThreads = 256;
constexpr int kRowsPerBlock = 4;

__device__ __forceinline__ uint32_t lstar_of(const double* lin, const double* thr, uint32_t r,
                                             uint32_t g, uint32_t b) {
    const double y =
        __dadd_rn(__dadd_rn(__dmul_rn(0.2126, lin[r]), __dmul_rn(0.7152, lin[g])),
                  __dmul_rn(0.0722, lin[b]));
    uint32_t v = 0;
#pragma unroll
    for (uint32_t step = 128; step > 0; step >>= 1)
        if (thr[v + step] <= y) v += step;
    return v;
}

// grid.x: row groups, grid.y: view (0 = left, 1 = right); `views` selects
// which views exist in this launch (bit 0 left, bit 1 right).
__global__ void __launch_bounds__(kThreads) k_lstar(Frame f, const LstarTables* __restrict__ tab,
                                                    int views, int do_hist, int vec) {
    __shared__ double lin[256];
    __shared__ double thr[256];
    __shared__ uint32_t hist[kThreads / 32][256];
    const int view = (views == 2) ? 1 : (int)blockIdx.y;
    const bool left = view == 0;
    const bool hist_on = do_hist && left;
    for (int i = threadIdx.x; i < 256; i += kThreads) {
        lin[i] = tab->linear[i];
        thr[i] = tab->thr[i];
    }
    if (hist_on)
        for (int i = threadIdx.x; i < (kThreads / 32) * 256; i += kThreads) (&hist[0][0])[i] = 0;
    __syncthreads();
    const uint8_t* __restrict__ rgb = left ? f.rgbL : f.rgbR;
    uint8_t* __restrict__ gray = left ? f.grayL : f.grayR;
    uint32_t* myh = hist[threadIdx.x >> 5];
    const int y0 = blockIdx.x * kRowsPerBlock;
    for (int y = y0; y < min(y0 + kRowsPerBlock, f.H); ++y) {
        const uint8_t* src = rgb + (size_t)y * f.W * 3;
        uint8_t* dst = gray + (size_t)y * f.P;
        if (vec) {
            // 16 pixels = 48 bytes = 3 x uint4 per thread
            for (int x = threadIdx.x * 16; x < f.W; x += kThreads * 16) {
                const uint4* s4 = reinterpret_cast<const uint4*>(src + (size_t)x * 3);
                uint4 a = __ldcs(s4), b = __ldcs(s4 + 1), c = __ldcs(s4 + 2);
                const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w,
                                        c.x, c.y, c.z, c.w};
                uint32_t out[4] = {0, 0, 0, 0};
#pragma unroll
                for (int p = 0; p < 16; ++p) {
                    const int o = p * 3;
                    const uint32_t r = (w[o >> 2] >> ((o & 3) * 8)) & 0xffu;
                    const uint32_t g = (w[(o + 1) >> 2] >> (((o + 1) & 3) * 8)) & 0xffu;
                    const uint32_t bb = (w[(o + 2) >> 2] >> (((o + 2) & 3) * 8)) & 0xffu;
                    const uint32_t v = lstar_of(lin, thr, r, g, bb);
                    out[p >> 2] |= v << ((p & 3) * 8);
                    if (hist_on) atomicAdd(&myh[v], 1u);
                }
                *reinterpret_cast<uint4*>(dst + x) = make_uint4(out[0], out[1], out[2], out[3]);
            }
        } else {
            for (int x = threadIdx.x; x < f.W; x += kThreads) {
                const uint8_t* p = src + (size_t)x * 3;
                const uint32_t v = lstar_of(lin, thr, p[0], p[1], p[2]);
                dst[x] = (uint8_t)v;
                if (hist_on) atomicAdd(&myh[v], 1u);
            }
        }
    }
    if (hist_on) {
        __syncthreads();
        for (int v = threadIdx.x; v < 256; v += kThreads) {
            uint32_t s = 0;
#pragma unroll
            for (int wi = 0; wi < kThreads / 32; ++wi) s += hist[wi][v];
            if (s) atomicAdd(&f.sc->hist[v], (unsigned long long)s);
        }
    }
}

// Histogram of an arbitrary pitched gray plane (stage entry build_histogram).
__global__ void __launch_bounds__(kThreads) k_hist(Frame f, const uint8_t* __restrict__ gray) {
    __shared__ uint32_t hist[kThreads / 32][256];
    for (int i = threadIdx.x; i < (kThreads / 32) * 256; i += kThreads) (&hist[0][0])[i] = 0;
    __syncthreads();
    uint32_t* myh = hist[threadIdx.x >> 5];
    for (int y = blockIdx.x; y < f.H; y += gridDim.x) {
        const uint8_t* row = gray + (size_t)y * f.P;
        for (int x = threadIdx.x; x < f.W; x += kThreads) atomicAdd(&myh[row[x]], 1u);
    }
    __syncthreads();
    for (int v = threadIdx.x; v < 256; v += kThreads) {
        uint32_t s = 0;
        for (int wi = 0; wi < kThreads / 32; ++wi) s += hist[wi][v];
        if (s) atomicAdd(&f.sc->hist[v], (unsigned long long)s);
    }
}

// labels[i] = bin_assignment[gray[i]]  (segmentation.cpp:146-155)
__global__ void k_assign(Frame f, const uint8_t* __restrict__ gray, uint16_t* __restrict__ out) {
    __shared__ uint16_t tab[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = f.sc->assign16[i];
    __syncthreads();
    const long long n = f.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        out[i] = tab[gray[(size_t)y * f.P + x]];
    }
}

}  // namespace

void launch_lightness(const Frame& f, const LstarTables* dtab, bool left, bool right, bool hist,
                      cudaStream_t st) {
    if (f.N == 0) return;
    const int views = (left && right) ? 3 : (left ? 1 : 2);
    const dim3 grid((f.H + kRowsPerBlock - 1) / kRowsPerBlock, views == 3 ? 2 : 1);
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(left ? f.rgbL : f.rgbR) |
          reinterpret_cast<uintptr_t>(right ? f.rgbR : f.rgbL)) & 15) == 0;
    const int vec = (f.W % 16 == 0) && aligned;
    k_lstar<<<grid, kThreads, 0, st>>>(f, dtab, views, hist ? 1 : 0, vec);
}

void launch_histogram(const Frame& f, const uint8_t* gray, cudaStream_t st) {
    if (f.N == 0) return;
    k_hist<<<std::min(f.H, 148 * 4), kThreads, 0, st>>>(f, gray);
}

void launch_assign(const Frame& f, const uint8_t* gray, uint16_t* out, cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 16);
    k_assign<<<(int)blocks, 256, 0, st>>>(f, gray, out);
}

}  // namespace stk
