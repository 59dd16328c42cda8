// Scratch probe: which u8/u16 TMA configurations run on this B200?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2001_07809_b200/csrc/stk_device.cuh"
using namespace stk;
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int bytes, int c0, int r0, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, bytes); tma_load_2d(sm, &m, &bar, c0, r0); }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) { unsigned s = 0; for (int i = 0; i < bytes; ++i) s += sm[i]; *out = s; }
}
int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  EncFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  uint8_t* buf; cudaMalloc(&buf, 1 << 22); cudaMemset(buf, 1, 1 << 22);
  unsigned* out; cudaMalloc(&out, 4);
  struct C { int esz, W, H, pitch, bw, bh, c0, r0; } cs[] = {
    {2, 450, 375, 1024, 144, 38, -8, -3}, {1, 450, 375, 512, 144, 38, -8, -3}, {1, 450, 375, 512, 144, 38, 8, 3},
    {1, 450, 375, 512, 128, 9, 0, 0}, {1, 512, 375, 512, 128, 8, 0, 0}, {1, 450, 375, 512, 64, 8, 0, 0},
    {1, 450, 375, 512, 16, 8, 0, 0}, {2, 450, 375, 1024, 64, 8, 0, 0},
    {1, 450, 375, 512, 128, 9, -20, -4}, {1, 450, 375, 512, 256, 8, 0, 0}, {1, 450, 375, 512, 160, 8, 0, 0},
    {1, 450, 375, 512, 144, 8, 0, 0}, {1, 450, 375, 512, 128, 21, -138, -10}, {1, 450, 375, 512, 192, 8, 0, 0},
    {1, 450, 375, 512, 32, 8, -5, -3}, {1, 450, 375, 512, 48, 8, 0, 0}};
  int i = atoi(argv[1]);
  auto& c = cs[i];
  CUtensorMap m;
  cuuint64_t gd[2] = {(cuuint64_t)c.W, (cuuint64_t)c.H}, gs[1] = {(cuuint64_t)c.pitch};
  cuuint32_t bd[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh}, es[2] = {1, 1};
  CUresult r = enc(&m, c.esz == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, buf, gd, gs, bd, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = c.bw * c.bh * c.esz;
  k<<<1, 32, bytes>>>(m, bytes, c.c0, c.r0, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h = 0;
  if (e == cudaSuccess) cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("case %d esz %d box %dx%d at (%d,%d): enc %d -> %s sum %u\n", i, c.esz, c.bw, c.bh, c.c0, c.r0, (int)r, cudaGetErrorString(e), h);
  return 0;
}
