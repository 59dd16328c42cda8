// PCIe copy-bandwidth probe: H2D / D2H alone and both at once (two streams),
// for host buffers from cudaMallocHost vs cudaHostAlloc(WriteCombined), and
// with the copies split into chunks over several streams.
#include <cstdio>
#include <cuda_runtime.h>

static float run(void (*fn)(void**), void** a, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    fn(a); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) fn(a);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}
static size_t N = 256ull << 20;
static int nchunk = 1;
static cudaStream_t s[8];
static void h2d(void** a) {
    for (int c = 0; c < nchunk; ++c)
        cudaMemcpyAsync((char*)a[1] + c * (N / nchunk), (char*)a[0] + c * (N / nchunk), N / nchunk, cudaMemcpyHostToDevice, s[c % 4]);
    for (int i = 0; i < 4; ++i) cudaStreamSynchronize(s[i]);
}
static void d2h(void** a) {
    for (int c = 0; c < nchunk; ++c)
        cudaMemcpyAsync((char*)a[2] + c * (N / nchunk), (char*)a[3] + c * (N / nchunk), N / nchunk, cudaMemcpyDeviceToHost, s[4 + c % 4]);
    for (int i = 4; i < 8; ++i) cudaStreamSynchronize(s[i]);
}
static void both(void** a) {
    for (int c = 0; c < nchunk; ++c) {
        cudaMemcpyAsync((char*)a[1] + c * (N / nchunk), (char*)a[0] + c * (N / nchunk), N / nchunk, cudaMemcpyHostToDevice, s[c % 4]);
        cudaMemcpyAsync((char*)a[2] + c * (N / nchunk), (char*)a[3] + c * (N / nchunk), N / nchunk, cudaMemcpyDeviceToHost, s[4 + c % 4]);
    }
    for (int i = 0; i < 8; ++i) cudaStreamSynchronize(s[i]);
}
int main() {
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    void *hp, *hwc, *hout, *d1, *d2;
    cudaMallocHost(&hp, N); cudaHostAlloc(&hwc, N, cudaHostAllocWriteCombined); cudaMallocHost(&hout, N);
    cudaMalloc(&d1, N); cudaMalloc(&d2, N);
    for (int wc = 0; wc < 2; ++wc)
        for (int ch : {1, 4, 16}) {
            nchunk = ch;
            void* a[4] = {wc ? hwc : hp, d1, hout, d2};
            const double gb = N / 1e9;
            printf("%s chunks %2d: H2D %.1f GB/s, D2H %.1f GB/s, duplex %.1f GB/s each way\n", wc ? "WC    " : "pinned", ch,
                   gb / (run(h2d, a, 5) * 1e-3), gb / (run(d2h, a, 5) * 1e-3), gb / (run(both, a, 5) * 1e-3));
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
