// Throughput probe: which pipe do K1's instructions use?  Each kernel runs a
// long dependent-free loop of one instruction kind on all SMs; time per
// instruction per SM tells the pipe rate.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k_fadd_rn(float* o, float a) {
    float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int n = 0; n < N; ++n)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fadd_rn(x[i], a);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd_rz(float* o, float a) {
    float x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int n = 0; n < N; ++n)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fadd_rz(x[i], a);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd2_rz(float* o, float a) {
    unsigned long long x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    const unsigned long long b = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
    for (int n = 0; n < N; ++n)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("add.rz.f32x2 %0, %0, %1;" : "+l"(x[i]) : "l"(b));
    unsigned long long s = 0; for (int i = 0; i < 8; ++i) s += x[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void k_shf64(float* o, float a) {
    uint32_t x[8]; for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    const uint32_t y = __float_as_uint(a);
    for (int n = 0; n < N; ++n)
#pragma unroll
        for (int i = 0; i < 8; ++i) { unsigned long long t = ((unsigned long long)y << 32) | x[i]; x[i] = (uint32_t)(t >> (n & 31)); }
    uint32_t s = 0; for (int i = 0; i < 8; ++i) s += x[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_atoms(float* o, float a) {
    __shared__ uint32_t h[32][256];
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t v = threadIdx.x * 2654435761u;
    for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { atomicAdd(&h[threadIdx.x >> 5][(v >> (8 * (i & 3))) & 255], 1u); v = v * 1664525u + 1013904223u; }
    }
    __syncthreads();
    o[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x >> 5][threadIdx.x & 255];
}
template <typename K>
void run(const char* name, K k, float* o) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<148 * 2, 1024>>>(o, 1.0f);
    cudaEventRecord(a);
    k<<<148 * 2, 1024>>>(o, 1.0f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double inst = 148.0 * 2 * 32 * (double)N * 8;  // warp-instructions
    printf("%-10s %8.3f ms  %.2f warp-inst/clk/SM (at 1.965 GHz)\n", name, ms, inst / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
    float* o; cudaMalloc(&o, 148 * 2 * 1024 * 4);
    run("fadd_rn", k_fadd_rn, o); run("fadd_rz", k_fadd_rz, o); run("fadd2_rz", k_fadd2_rz, o);
    run("shf64", k_shf64, o); run("atoms", k_atoms, o);
    return 0;
}
