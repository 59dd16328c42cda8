// K5 sad_match -- winner-takes-all SAD block matching on the compacted list of
// boundary pixels only (reference: stereo.cpp:12-28, 62-102).
//
// K5a sad_list (the per-pixel design): persistent CTAs claim row-tiles
//   (row y, 128 columns) in order.  For a tile with list entries, rows
//   [y-h, y+h] of the left view (columns x0-h .. x0+127+h) and of the right
//   view (columns x0-h-D .. x0+127+h) arrive through cp.async.bulk.tensor
//   boxes of 128x w bytes and are repacked into linear shared-memory rows.
//   One warp per boundary pixel, lanes = disparities (d = lane + 32 j); each
//   lane accumulates byte SADs four at a time with vabsdiff4.add on
//   funnel-shift realigned words; the winner is a warp __reduce_min over the
//   key (cost << 10 | d), which yields "strict <, ties to the smallest d"
//   (stereo.cpp:90-97) for free.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBox = 128;  // TMA box width (bytes / columns)

__device__ __forceinline__ uint32_t vsad4_acc(uint32_t a, uint32_t b, uint32_t acc) {
    uint32_t r;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(acc));
    return r;
}

__device__ __forceinline__ uint32_t ld_unaligned(const uint8_t* row, int off) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(row + (off & ~3));
    return __funnelshift_r(p[0], p[1], (off & 3) * 8);
}

template <int MAXJ>
__global__ void __launch_bounds__(kThreads) k_sad_list(const __grid_constant__ CUtensorMap tmL,
                                                       const __grid_constant__ CUtensorMap tmR,
                                                       Frame f) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ int s_tile;
    const int w = f.window, h = f.hw, D = f.D, W = f.W;
    // 8-bit TMA boxes must start on a 16-byte column boundary, so each view's
    // box run starts at (first needed column) & ~15 and the windows are read
    // at that offset (offL/offR, constant because x0 is a multiple of 128).
    const int nbL = (15 + kRowTile + 2 * h + kBox - 1) / kBox;
    const int nbR = (15 + kRowTile + 2 * h + D + kBox - 1) / kBox;
    const int offL = (-h) & 15, offR = (-h - D) & 15;
    const int LP = nbL * kBox + 16, RP = nbR * kBox + 16;  // linear row pitches (+ slack)
    uint8_t* stage = smem;                                   // (nbL+nbR) * w * kBox
    uint8_t* Ll = stage + (size_t)(nbL + nbR) * w * kBox;    // w * LP
    uint8_t* Rl = Ll + (size_t)w * LP;                       // w * RP
    const int nw = (w + 3) >> 2;
    const uint32_t tail = (w & 3) ? (0xffffffffu >> (32 - 8 * (w & 3))) : 0xffffffffu;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmL);
        tma_prefetch_desc(&tmR);
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    while (true) {
        __syncthreads();  // everyone has read the previous s_tile
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(&f.sc->ctr[LB_SAD], 1u);
        __syncthreads();
        const int t = s_tile;
        if (t >= f.n_tiles) break;
        const uint32_t e0 = f.tile_off[t], e1 = f.tile_off[t + 1];
        if (e0 == e1) continue;  // uniform: every thread sees the same tile
        const int y = t / f.TX, x0 = (t % f.TX) * kRowTile;
        if (threadIdx.x == 0) {
            mbar_expect_tx(&bar, (uint32_t)((nbL + nbR) * w * kBox));
            for (int i = 0; i < nbL; ++i)
                tma_load_2d(stage + (size_t)i * w * kBox, &tmL, &bar, x0 - h - offL + i * kBox,
                            y - h);
            for (int i = 0; i < nbR; ++i)
                tma_load_2d(stage + (size_t)(nbL + i) * w * kBox, &tmR, &bar,
                            x0 - h - D - offR + i * kBox, y - h);
        }
        mbar_wait(&bar, phase);
        phase ^= 1;
        // repack boxes [box][row][128] -> linear rows
        for (int i = threadIdx.x; i < (nbL + nbR) * w * (kBox / 4); i += kThreads) {
            const int bx = i / (w * (kBox / 4)), rem = i % (w * (kBox / 4));
            const int r = rem / (kBox / 4), c4 = rem % (kBox / 4);
            const uint32_t v = reinterpret_cast<const uint32_t*>(stage)[i];
            if (bx < nbL)
                reinterpret_cast<uint32_t*>(Ll + (size_t)r * LP + bx * kBox)[c4] = v;
            else
                reinterpret_cast<uint32_t*>(Rl + (size_t)r * RP + (bx - nbL) * kBox)[c4] = v;
        }
        __syncthreads();
        for (uint32_t e = e0 + wid; e < e1; e += kWarps) {
            const uint32_t code = f.list[e];
            const int x = (int)(code & 0xffffu);
            const int lx = x - x0 + offL;          // L window starts at Ll col lx
            const int dl = min(D, x - h);
            uint32_t cost[MAXJ];
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) cost[j] = 0;
            for (int r = 0; r < w; ++r) {
                const uint8_t* lrow = Ll + (size_t)r * LP;
                const uint8_t* rrow = Rl + (size_t)r * RP;
                uint32_t lw[16];
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (k < nw) lw[k] = ld_unaligned(lrow, lx + 4 * k) & (k == nw - 1 ? tail : ~0u);
#pragma unroll
                for (int j = 0; j < MAXJ; ++j) {
                    const int d = lane + 32 * j;
                    if (d > dl) continue;
                    const int ro = lx - offL - d + D + offR;  // R window of x-d in Rl
                    uint32_t acc = cost[j];
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (k < nw)
                            acc = vsad4_acc(lw[k],
                                            ld_unaligned(rrow, ro + 4 * k) & (k == nw - 1 ? tail : ~0u),
                                            acc);
                    cost[j] = acc;
                }
            }
            uint32_t key = 0xffffffffu;
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) {
                const int d = lane + 32 * j;
                if (d <= dl) key = min(key, (cost[j] << 10) | (uint32_t)d);
            }
            key = __reduce_min_sync(0xffffffffu, key);
            if (lane == 0) f.sparse[(size_t)y * W + x] = (int16_t)(key & 1023u);
        }
    }
}

template <int MAXJ>
void run_list(const Frame& f, const CUtensorMap* tmL, const CUtensorMap* tmR, cudaStream_t st) {
    const size_t sm = sad_list_smem_bytes(f.window, f.D);
    cudaFuncSetAttribute(k_sad_list<MAXJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sad_list<MAXJ>, kThreads, sm);
    k_sad_list<MAXJ><<<f.sms * std::max(per_sm, 1), kThreads, sm, st>>>(*tmL, *tmR, f);
}

// K5w sad_wide: any window and disparity range (the reference accepts any odd
// window >= 1 and any max_disparity >= 0, stereo.cpp:49-57).  One warp per
// list entry, lanes = disparities d = lane + 32 j (ascending per lane, strict
// <), exact u32 sums (wrapping like the reference's uint32_t) of byte SADs four
// at a time from the pitched gray planes (L2-resident); the winner is the warp
// minimum of the 64-bit key (cost << 32 | d): ties to the smallest d.
__global__ void __launch_bounds__(kThreads) k_sad_wide(Frame f) {
    const int w = f.window, h = f.hw, D = f.D;
    const int nw = (w + 3) >> 2;
    const uint32_t tail = (w & 3) ? (0xffffffffu >> (32 - 8 * (w & 3))) : 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const long long n = f.sc->n_list;
    for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; e < n;
         e += ((long long)gridDim.x * blockDim.x) >> 5) {
        const uint32_t code = f.list[e];
        const int x = (int)(code & 0xffffu), y = (int)(code >> 16);
        const int dl = min(D, x - h);
        unsigned long long best = ~0ull;
        for (int d = lane; d <= dl; d += 32) {
            uint32_t cost = 0;
            for (int r = 0; r < w; ++r) {
                const uint8_t* lrow = f.grayL + (size_t)(y - h + r) * f.P;
                const uint8_t* rrow = f.grayR + (size_t)(y - h + r) * f.P;
                for (int k = 0; k < nw; ++k) {
                    const uint32_t m = k == nw - 1 ? tail : 0xffffffffu;
                    cost = vsad4_acc(ld_unaligned(lrow, x - h + 4 * k) & m,
                                     ld_unaligned(rrow, x - d - h + 4 * k) & m, cost);
                }
            }
            const unsigned long long key = ((unsigned long long)cost << 32) | (uint32_t)d;
            best = key < best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
            best = v < best ? v : best;
        }
        if (lane == 0) f.sparse[(size_t)y * f.W + x] = (int16_t)(uint32_t)best;
    }
}

// sad_cost for one (x, y, d) (stereo.cpp:12-28): one warp, lanes stride the
// window rows, exact u32 sum.
__global__ void k_sad_cost(Frame f, int x, int y, int d, uint32_t* out) {
    const int h = f.hw, w = f.window;
    uint32_t s = 0;
    for (int r = threadIdx.x; r < w; r += 32) {
        const uint8_t* l = f.grayL + (size_t)(y - h + r) * f.P + (x - h);
        const uint8_t* rr = f.grayR + (size_t)(y - h + r) * f.P + (x - d - h);
        for (int i = 0; i < w; ++i) s += (uint32_t)abs((int)l[i] - (int)rr[i]);
    }
    s = __reduce_add_sync(0xffffffffu, s);
    if (threadIdx.x == 0) *out = s;
}

}  // namespace

void launch_sad_cost(const Frame& f, int x, int y, int d, uint32_t* out, cudaStream_t st) {
    k_sad_cost<<<1, 32, 0, st>>>(f, x, y, d, out);
}

size_t sad_list_smem_bytes(int window, int D) {
    const int h = window / 2;
    const int nbL = (15 + kRowTile + 2 * h + kBox - 1) / kBox;
    const int nbR = (15 + kRowTile + 2 * h + D + kBox - 1) / kBox;
    return (size_t)(nbL + nbR) * window * kBox + (size_t)window * (nbL * kBox + 16) +
           (size_t)window * (nbR * kBox + 16);
}

// the TMA list kernel's reach: 16 words per window row, d in 10 key bits,
// its staged rows in shared memory
static bool list_fits(const Frame& f) {
    return f.window <= 63 && f.D <= 1023 && sad_list_smem_bytes(f.window, f.D) <= 227 * 1024;
}

bool sad_uses_list(const Frame& f, int kernel) {
    if (f.N == 0 || f.W < f.window || f.H < f.window) return false;
    if ((kernel == SAD_AUTO || kernel == SAD_WS) && launch_sad_ws(f, nullptr, true)) return false;
    if (kernel != SAD_LIST && launch_sad_strip(f, nullptr, true)) return false;
    return true;
}

void launch_sad(const Frame& f, int kernel, const CUtensorMap* tmL, const CUtensorMap* tmR,
                cudaStream_t st) {
    if (f.N == 0 || f.W < f.window || f.H < f.window) return;
    if ((kernel == SAD_AUTO || kernel == SAD_WS) && launch_sad_ws(f, st)) return;
    if (kernel != SAD_LIST && launch_sad_strip(f, st)) return;
    if (!list_fits(f)) {
        k_sad_wide<<<f.sms * 8, kThreads, 0, st>>>(f);
        return;
    }
    const int J = (f.D + 1 + 31) / 32;
    if (J <= 1) run_list<1>(f, tmL, tmR, st);
    else if (J <= 2) run_list<2>(f, tmL, tmR, st);
    else if (J <= 4) run_list<4>(f, tmL, tmR, st);
    else if (J <= 8) run_list<8>(f, tmL, tmR, st);
    else if (J <= 16) run_list<16>(f, tmL, tmR, st);
    else run_list<32>(f, tmL, tmR, st);
}

}  // namespace stk
