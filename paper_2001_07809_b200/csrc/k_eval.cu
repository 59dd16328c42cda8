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

// VABSDIFF4 issue-rate probe (the match stage's brute-force
// ALU ceiling is microbenchmarked on the box): 8 independent chains per
// thread, 32 VABSDIFF4 per loop trip, no memory traffic.
__global__ void __launch_bounds__(256) k_vabsdiff4_probe(uint32_t seed, int iters, uint32_t* out) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (2 * i + 1) + threadIdx.x;
        b[i] = (seed ^ 0x9e3779b9u) * (i + 3) + blockIdx.x;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __vabsdiffu4(a[i], b[i]);
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= a[i];
    if (x == seed) out[0] = x;  // keeps the chains alive; practically never taken
}

}  // namespace

double probe_vabsdiff4_rate(int sms, uint32_t* scratch, cudaStream_t st) {
    const int blocks = sms * 8, iters = 8192;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_vabsdiff4_probe<<<blocks, 256, 0, st>>>(12345u, iters, scratch);  // warm-up (clocks up)
    float best = 0.f;
    for (int rep = 0; rep < 3; ++rep) {  // best of 3
        cudaEventRecord(e0, st);
        k_vabsdiff4_probe<<<blocks, 256, 0, st>>>(12345u, iters, scratch);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms > 0.f && (best == 0.f || ms < best)) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess || best <= 0.f) return 0.0;
    const double ops = (double)blocks * 256 * iters * 32;  // VABSDIFF4 instructions (4 byte-ADs each)
    return ops / (best * 1e-3);
}

void launch_bad_pixel(const int16_t* comp, const int16_t* truth, long long n, double delta,
                      unsigned long long* out, cudaStream_t st) {
    if (n <= 0) return;
    const int blocks = (int)std::min<long long>((n / 8 + 255) / 256 + 1, 148 * 8);
    k_bad_pixel<<<blocks, 256, 0, st>>>(comp, truth, n, delta, out);
}

}  // namespace stk
