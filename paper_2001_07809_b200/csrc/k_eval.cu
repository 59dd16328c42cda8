// K9 -- evaluation on the GPU (reference: evaluate.cpp).
//
//   bad_pixel_rate (evaluate.cpp:17-74): pixels known in both maps are
//   compared; bad iff |computed - truth| > delta_d.  One pass, 8 int16 pairs
//   per thread-step with 16-byte loads, warp + block reductions, two u64
//   atomics per block.
//   dense_sad_baseline (evaluate.cpp:92-135) is match_boundary_pixels with
//   every pixel in the mask (the reference's own test asserts the equality,
//   test_evaluate.cpp:125-143); its stage entry fills the mask plane and runs
//   the SAD kernels.
#include "stk_device.cuh"

namespace stk {

namespace {

__global__ void __launch_bounds__(256) k_bad_pixel(const int16_t* __restrict__ comp,
                                                   const int16_t* __restrict__ truth, long long n,
                                                   double delta, unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sc[8], sb[8];
    unsigned long long cmp = 0, bad = 0;
    auto one = [&](int c, int t) {
        if (c < 0 || t < 0) return;
        ++cmp;
        const int d = c >= t ? c - t : t - c;
        if ((double)d > delta) ++bad;
    };
    const long long n8 = (reinterpret_cast<uintptr_t>(comp) | reinterpret_cast<uintptr_t>(truth)) & 15 ? 0 : n / 8;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += stride) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4*>(comp) + i);
        const uint4 b = __ldcs(reinterpret_cast<const uint4*>(truth) + i);
        const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            one((int16_t)(wa[k] & 0xffffu), (int16_t)(wb[k] & 0xffffu));
            one((int16_t)(wa[k] >> 16), (int16_t)(wb[k] >> 16));
        }
    }
    for (long long i = 8 * n8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        one(comp[i], truth[i]);
    for (int o = 16; o > 0; o >>= 1) {
        cmp += __shfl_xor_sync(0xffffffffu, cmp, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sc[threadIdx.x >> 5] = cmp;
        sb[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tc = 0, tb = 0;
        for (int i = 0; i < 8; ++i) tc += sc[i], tb += sb[i];
        if (tc) atomicAdd(out, tc);
        if (tb) atomicAdd(out + 1, tb);
    }
}

}  // namespace

void launch_bad_pixel(const int16_t* comp, const int16_t* truth, long long n, double delta,
                      unsigned long long* out, cudaStream_t st) {
    if (n <= 0) return;
    const int blocks = (int)std::min<long long>((n / 8 + 255) / 256 + 1, 148 * 8);
    k_bad_pixel<<<blocks, 256, 0, st>>>(comp, truth, n, delta, out);
}

}  // namespace stk
