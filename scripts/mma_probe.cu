// Microbenchmark: legacy mma.sync (HMMA) throughput on this GPU, f16 inputs,
// f32 accumulate, m16n8k16; and FFMA2 for comparison.  Prints MAC/clk/SM.
#include <cstdio>
#include <cuda_fp16.h>

__global__ void k_hmma(float* out, int iters) {
    unsigned a0 = 0x3c003c00u ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0x3c003c00u, b1 = b0 + 7;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters) {
    unsigned long long a[8], w = 0x3f8000003f800000ull ^ threadIdx.x;
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[j]) : "l"(w), "l"(w));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s ^= a[j];
    if (s == 12345) out[threadIdx.x] = (float)s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4096);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_hmma<<<sms, 32 * warps>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double macs = (double)sms * warps * iters * 8 * 16 * 8 * 16;
            if (rep) printf("HMMA warps/SM %2d: %.3f ms, %.0f MAC/clk/SM (at %d MHz), %.1f TFLOP/s\n", warps, ms,
                            macs / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, 2 * macs / (ms * 1e-3) / 1e12);
            cudaEventRecord(e0);
            k_ffma2<<<sms, 32 * warps>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double fmas = (double)sms * warps * 32 * iters * 8 * 2;
            if (rep) printf("FFMA2 warps/SM %2d: %.3f ms, %.0f FMA/clk/SM\n", warps, ms, fmas / (ms * 1e-3) / sms / (clk * 1e3));
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
