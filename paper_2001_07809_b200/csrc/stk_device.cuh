// stk_device.cuh -- device helpers shared by the kernels: TMA + mbarrier
// wrappers (inline PTX, sm_100a), warp/block reductions, and the single-pass
// decoupled look-back used by every ordered stream compaction.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "stk_internal.cuh"

namespace stk {

// ------------------------------------------------------------------ TMA ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1-D bulk copy global -> shared (cp.async.bulk, SASS UBLKCP); 16-byte aligned
// addresses, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Named CTA barriers (producer/consumer hand-off between warp groups).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 2-D tiled TMA load (cp.async.bulk.tensor) of box {c0.., r0..} into smem.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int r0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ------------------------------------------------------------ reductions ----
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
    return __reduce_add_sync(0xffffffffu, v);
}

template <int NT>
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long* sh) {
    // sh: >= NT/32 entries
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) t += sh[i];
    return t;  // valid in thread 0 only
}

// ------------------------------------------------ decoupled look-back scan --
// Status word: bits 63..62 = flag (0 none, 1 aggregate, 2 inclusive prefix),
// bits 31..0 = value.  Chunks are claimed in order through an atomic counter so
// every predecessor of a spinning chunk is already resident.
__device__ __forceinline__ void lb_publish(unsigned long long* p, unsigned long long flag,
                                           uint32_t val) {
    const unsigned long long v = (flag << 62) | val;
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ALL 32 lanes of one warp: returns (on every lane) the exclusive
// prefix of chunk `c` whose own total is `agg`, and publishes the inclusive
// prefix.  The warp polls 32 predecessors per round, so an aggregate-only
// run of predecessors costs one round trip per 32 chunks.
__device__ __forceinline__ uint32_t lb_exclusive_warp(unsigned long long* status, int c,
                                                      uint32_t agg) {
    const int lane = threadIdx.x & 31;
    if (c == 0) {
        if (lane == 0) lb_publish(status, 2ull, agg);
        return 0;
    }
    if (lane == 0) lb_publish(status + c, 1ull, agg);
    uint32_t excl = 0;
    int j = c - 1;
    while (true) {
        const int idx = j - lane;
        const unsigned long long v = idx >= 0 ? lb_load(status + idx) : (2ull << 62);
        const unsigned flag = (unsigned)(v >> 62);
        const unsigned incl = __ballot_sync(0xffffffffu, flag == 2u);
        const unsigned zero = __ballot_sync(0xffffffffu, flag == 0u);
        const int first = incl ? __ffs(incl) - 1 : 32;
        const unsigned upto = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
        if (zero & upto) continue;  // a predecessor we need has not published yet
        const uint32_t val = lane <= first ? (uint32_t)(v & 0xffffffffu) : 0u;
        excl += __reduce_add_sync(0xffffffffu, val);
        if (first < 32) break;
        j -= 32;
    }
    if (lane == 0) lb_publish(status + c, 2ull, excl + agg);
    return excl;
}

// Called by ONE thread: returns the exclusive prefix of chunk `c` whose own
// total is `agg`, and publishes the inclusive prefix.
__device__ __forceinline__ uint32_t lb_exclusive(unsigned long long* status, int c, uint32_t agg) {
    if (c == 0) {
        lb_publish(status, 2ull, agg);
        return 0;
    }
    lb_publish(status + c, 1ull, agg);
    uint32_t excl = 0;
    int j = c - 1;
    while (true) {
        unsigned long long v = lb_load(status + j);
        const unsigned long long flag = v >> 62;
        if (flag == 0) continue;  // predecessor not published yet
        excl += static_cast<uint32_t>(v & 0xffffffffu);
        if (flag == 2) break;
        --j;
    }
    lb_publish(status + c, 2ull, excl + agg);
    return excl;
}

}  // namespace stk
