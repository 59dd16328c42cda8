// K4 -- connected components, prune, anchors and boundary-pixel compaction,
// all on the device with no host round trip (reference: boundary.cpp:87-195,
// pipeline.cpp:92-94).
//
//   K4a ccl_local    32x32 tile union-find in shared memory (atomicMin union,
//                    path compression), min-index roots.
//   K4b ccl_merge    tile-border pixels unite across tiles in global memory
//                    (lock-free atomicMin union on raster indices).
//   K4c ccl_flatten  every pixel -> its root (= min raster index of its
//                    component); component sizes by warp-aggregated atomics.
//   K4d ccl_roots    ordered compaction of roots (decoupled look-back):
//                    canonical label = rank of the root in raster order, which
//                    is exactly the reference's discovery order; size
//                    histogram for the prune.
//   K4e prune_select counting-sort form of the reference's by_size walk.
//   K4f prune_mark   marks removed components (rank among size-s* roots).
//   K4g apply        prune + border anchors + window filter + warp-ballot
//                    ordered compaction into the raster-ordered boundary list,
//                    the matchable bit-mask and per-row-tile list offsets.
//
// Prune equivalence (boundary.cpp:150-178): by_size orders (size, label);
// the walk removes a prefix while removed+size <= budget, i.e. <= B =
// floor(budget).  With CS(s) = pixels in components of size <= s, let s* be
// the smallest size with CS(s*) > B: every component smaller than s* goes,
// plus the first q = floor((B - CS(s*-1)) / s*) size-s* components in label
// order.  Components larger than B+1 can never be removed, so the size
// histogram only needs bins 1..B+1.
#include "stk_device.cuh"

namespace stk {

namespace {

constexpr int CT = 32;  // CCL tile side

// ------------------------------------------------------------ union-find --
__device__ __forceinline__ int sfind(volatile int* p, int x) {
    int q = p[x];
    while (q != x) {
        x = q;
        q = p[x];
    }
    return x;
}

__device__ __forceinline__ void sunite(int* p, int a, int b) {
    while (true) {
        a = sfind(p, a);
        b = sfind(p, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(&p[b], a);
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ int gfind(const int* p, int x) {
    int q = __ldcg(p + x);
    while (q != x) {
        x = q;
        q = __ldcg(p + x);
    }
    return x;
}

__device__ __forceinline__ void gunite(int* p, int a, int b) {
    while (true) {
        a = gfind(p, a);
        b = gfind(p, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(p + b, a);
        if (old == b) return;
        b = old;
    }
}

__device__ __forceinline__ unsigned long long budget_of(const Frame& f) {
    // boundary.cpp:156: fraction * double(mask.count()); integer sizes compare
    // <= budget  <=>  <= floor(budget)
    return (unsigned long long)floor(__dmul_rn(f.frac, (double)f.sc->refined_count));
}

// ----------------------------------------------------------------- K4a ----
__global__ void __launch_bounds__(256) k_ccl_local(Frame f) {
    __shared__ int lp[CT * CT];
    const int x0 = blockIdx.x * CT, y0 = blockIdx.y * CT;
    const int tid = threadIdx.x;
    for (int i = tid; i < CT * CT; i += 256) {
        const int x = x0 + (i & (CT - 1)), y = y0 + i / CT;
        const bool set = x < f.W && y < f.H && f.mref[(size_t)y * f.P + x];
        lp[i] = set ? i : -1;
    }
    // zero the size histogram bins the prune will use (0..B+1)
    {
        const unsigned long long B = budget_of(f);
        const long long nb = (long long)gridDim.x * gridDim.y;
        const long long bid = blockIdx.y * (long long)gridDim.x + blockIdx.x;
        for (long long s = bid * 256 + tid; s <= (long long)B + 1; s += nb * 256) f.szhist[s] = 0;
        if (bid == 0 && tid == 0) f.sc->budget = B;
    }
    __syncthreads();
    for (int i = tid; i < CT * CT; i += 256) {
        if (lp[i] < 0) continue;
        const int c = i & (CT - 1), r = i / CT;
        // backward Moore neighbours W, NW, N, NE
        if (c > 0 && lp[i - 1] >= 0) sunite(lp, i, i - 1);
        if (r > 0) {
            if (c > 0 && lp[i - CT - 1] >= 0) sunite(lp, i, i - CT - 1);
            if (lp[i - CT] >= 0) sunite(lp, i, i - CT);
            if (c < CT - 1 && lp[i - CT + 1] >= 0) sunite(lp, i, i - CT + 1);
        }
    }
    __syncthreads();
    int roots[CT * CT / 256];
#pragma unroll
    for (int k = 0; k < CT * CT / 256; ++k) {
        const int i = tid + k * 256;
        roots[k] = lp[i] >= 0 ? sfind(lp, i) : -1;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CT * CT / 256; ++k) {
        const int i = tid + k * 256;
        if (roots[k] < 0) continue;
        const int x = x0 + (i & (CT - 1)), y = y0 + i / CT;
        const int rx = x0 + (roots[k] & (CT - 1)), ry = y0 + roots[k] / CT;
        const int g = y * f.W + x, gr = ry * f.W + rx;
        f.par[g] = gr;
        if (gr == g) f.cnt[g] = 0;
    }
}

// ----------------------------------------------------------------- K4b ----
__global__ void __launch_bounds__(128) k_ccl_merge(Frame f) {
    const int x0 = blockIdx.x * CT, y0 = blockIdx.y * CT;
    const int t = threadIdx.x;
    int x, y;
    if (t < 32) {  // top row
        x = x0 + t;
        y = y0;
    } else if (t < 64) {  // left column
        x = x0;
        y = y0 + (t - 32);
    } else if (t < 96) {  // right column
        x = x0 + CT - 1;
        y = y0 + (t - 64);
    } else {
        return;
    }
    if (x >= f.W || y >= f.H || !f.mref[(size_t)y * f.P + x]) return;
    const int g = y * f.W + x;
    const int nx[4] = {x - 1, x - 1, x, x + 1}, ny[4] = {y, y - 1, y - 1, y - 1};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int qx = nx[k], qy = ny[k];
        if (qx < 0 || qx >= f.W || qy < 0) continue;
        if (qx / CT == blockIdx.x && qy / CT == blockIdx.y) continue;  // same tile: done in K4a
        if (!f.mref[(size_t)qy * f.P + qx]) continue;
        gunite(f.par, g, qy * f.W + qx);
    }
}

// ----------------------------------------------------------------- K4c ----
__global__ void __launch_bounds__(256) k_ccl_flatten(Frame f) {
    const int y = blockIdx.y;
    const int x = blockIdx.x * 256 + threadIdx.x;
    int r = -1;
    if (x < f.W && f.mref[(size_t)y * f.P + x]) {
        const int g = y * f.W + x;
        r = gfind(f.par, g);
        f.par[g] = r;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    if (r >= 0 && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
        atomicAdd(f.cnt + r, (unsigned)__popc(peers));
}

// ----------------------------------------------------------------- K4d ----
// Chunk = 8 row-tiles (one warp each, 128 pixels of one row, 4 per lane at
// x = seg*128 + j*32 + lane so ballots come out in raster order).
__global__ void __launch_bounds__(256) k_ccl_roots(Frame f, int write_rank) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* status = f.lb + LB_ROOTS * f.lb_stride;
    if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_ROOTS], 1u);
    __syncthreads();
    const int c = s_chunk;
    const int t = c * kTilesPerChunk + wid;
    uint32_t balls[4] = {0, 0, 0, 0};
    int gidx[4];
    if (t < f.n_tiles) {
        const int y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = seg * kRowTile + j * 32 + lane;
            gidx[j] = y * f.W + x;
            bool isroot = false;
            if (x < f.W && f.mref[(size_t)y * f.P + x]) isroot = f.par[gidx[j]] == gidx[j];
            balls[j] = __ballot_sync(0xffffffffu, isroot);
        }
    }
    const uint32_t wc = __popc(balls[0]) + __popc(balls[1]) + __popc(balls[2]) + __popc(balls[3]);
    if (lane == 0) wcount[wid] = wc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t agg = 0;
        for (int i = 0; i < 8; ++i) agg += wcount[i];
        const uint32_t excl = lb_exclusive(status, c, agg);
        s_excl = excl;
        if (c == f.n_chunks - 1) f.sc->n_roots = excl + agg;
    }
    __syncthreads();
    if (t >= f.n_tiles) return;
    uint32_t pos = s_excl;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    const unsigned long long B = f.sc->budget;
    const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (balls[j] >> lane & 1u) {
            const uint32_t p = pos + __popc(balls[j] & lanemask);
            f.roots[p] = gidx[j];
            if (write_rank) f.rank[gidx[j]] = (int)p;
            const uint32_t sz = f.cnt[gidx[j]];
            if (sz <= B + 1) atomicAdd(f.szhist + sz, 1u);
        }
        pos += __popc(balls[j]);
    }
}

// ----------------------------------------------------------------- K4e ----
__global__ void __launch_bounds__(1024) k_prune_select(Frame f) {
    __shared__ unsigned long long part[1024];
    DevScalars* sc = f.sc;
    const unsigned long long B = sc->budget;
    const long long L = (long long)B + 1;  // sizes 1..B+1
    const long long per = (L + 1023) / 1024;
    const long long s0 = 1 + threadIdx.x * per, s1 = min(s0 + per, L + 1);
    unsigned long long sum = 0;
    for (long long s = s0; s < s1; ++s) sum += (unsigned long long)s * f.szhist[s];
    part[threadIdx.x] = sum;
    __syncthreads();
    // inclusive scan (Hillis-Steele) over 1024 partials
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned long long v = threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    const unsigned long long before = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
    if (threadIdx.x == 0) {
        sc->s_star = B + 2;  // default: remove every size <= B+1, q = 0
        sc->q = 0;
    }
    __syncthreads();
    if (before <= B && part[threadIdx.x] > B) {  // exactly one thread
        unsigned long long cs = before;
        for (long long s = s0; s < s1; ++s) {
            const unsigned long long add = (unsigned long long)s * f.szhist[s];
            if (cs + add > B) {
                sc->s_star = (unsigned long long)s;
                sc->q = (B - cs) / (unsigned long long)s;
                break;
            }
            cs += add;
        }
    }
}

// ----------------------------------------------------------------- K4f ----
// Persistent: chunks of 1024 roots claimed in order; ordered rank of size-s*
// roots by decoupled look-back only matters when q > 0.
__global__ void __launch_bounds__(256) k_prune_mark(Frame f) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[8];
    const uint32_t C = f.sc->n_roots;
    const unsigned long long sst = f.sc->s_star, q = f.sc->q;
    unsigned long long* status = f.lb + LB_RANK * f.lb_stride;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_RANK], 1u);
        __syncthreads();
        const uint32_t c = s_chunk;
        if ((unsigned long long)c * 1024 >= C) return;
        uint32_t balls[4];
        int r[4];
        uint32_t sz[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t idx = c * 1024 + wid * 128 + j * 32 + lane;
            r[j] = idx < C ? f.roots[idx] : -1;
            sz[j] = r[j] >= 0 ? f.cnt[r[j]] : 0;
            balls[j] = __ballot_sync(0xffffffffu, r[j] >= 0 && sz[j] == sst);
        }
        uint32_t pos = 0;
        if (q > 0) {
            const uint32_t wc =
                __popc(balls[0]) + __popc(balls[1]) + __popc(balls[2]) + __popc(balls[3]);
            if (lane == 0) wcount[wid] = wc;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t agg = 0;
                for (int i = 0; i < 8; ++i) agg += wcount[i];
                s_excl = lb_exclusive(status, (int)c, agg);
            }
            __syncthreads();
            pos = s_excl;
            for (int i = 0; i < wid; ++i) pos += wcount[i];
        }
        const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (r[j] >= 0) {
                bool rm = sz[j] < sst;
                if (!rm && (balls[j] >> lane & 1u)) rm = pos + __popc(balls[j] & lanemask) < q;
                if (rm) f.cnt[r[j]] = sz[j] | kRemoved;
            }
            pos += __popc(balls[j]);
        }
    }
}

// ----------------------------------------------------------------- K4g ----
__global__ void __launch_bounds__(256) k_apply(Frame f, int use_prune, int anchors) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[8];
    __shared__ unsigned long long red[8], red2[8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* status = f.lb + LB_LIST * f.lb_stride;
    if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_LIST], 1u);
    __syncthreads();
    const int c = s_chunk;
    const int t = c * kTilesPerChunk + wid;
    const int m = f.hw, W = f.W, H = f.H;
    uint32_t balls[4] = {0, 0, 0, 0};
    uint32_t kept = 0;
    unsigned long long ops = 0;
    int y = 0, seg = 0;
    if (t < f.n_tiles) {
        y = t / f.TX;
        seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = seg * kRowTile + j * 32 + lane;
            bool keep = false, anc = false;
            if (x < W) {
                const size_t po = (size_t)y * f.P + x;
                const int g = y * W + x;
                if (f.mref[po]) keep = use_prune ? !(f.cnt[f.par[g]] & kRemoved) : true;
                anc = keep;
                if (anchors && (x == m || x == W - 1 - m) && y >= m && y <= H - 1 - m) anc = true;
                if (f.mprn) f.mprn[po] = keep;
                if (f.manc) f.manc[po] = anc;
                f.sparse[g] = -1;
            }
            kept += keep;
            const bool matchable = anc && y >= m && y < H - m && x >= m && x < W - m;
            balls[j] = __ballot_sync(0xffffffffu, matchable);
            if (matchable) ops += (unsigned long long)(min(f.D, x - m) + 1);
            if (lane == 0) f.mbits[(size_t)y * f.bits_words + seg * 4 + j] = balls[j];
        }
    }
    const uint32_t wc = __popc(balls[0]) + __popc(balls[1]) + __popc(balls[2]) + __popc(balls[3]);
    if (lane == 0) wcount[wid] = wc;
    unsigned long long kk = kept, oo = ops;
    for (int o = 16; o > 0; o >>= 1) {
        kk += __shfl_xor_sync(0xffffffffu, kk, o);
        oo += __shfl_xor_sync(0xffffffffu, oo, o);
    }
    if (lane == 0) {
        red[wid] = kk;
        red2[wid] = oo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t agg = 0;
        unsigned long long ka = 0, oa = 0;
        for (int i = 0; i < 8; ++i) {
            agg += wcount[i];
            ka += red[i];
            oa += red2[i];
        }
        const uint32_t excl = lb_exclusive(status, c, agg);
        s_excl = excl;
        if (ka) atomicAdd(&f.sc->pruned_count, ka);
        if (oa) atomicAdd(&f.sc->sad_ops, oa * (unsigned long long)(f.window * f.window));
        if (c == f.n_chunks - 1) {
            f.sc->n_list = excl + agg;
            f.sc->matched = excl + agg;
            f.tile_off[f.n_tiles] = excl + agg;
        }
    }
    __syncthreads();
    if (t >= f.n_tiles) return;
    uint32_t pos = s_excl;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    if (lane == 0) f.tile_off[t] = pos;
    const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (balls[j] >> lane & 1u) {
            const int x = seg * kRowTile + j * 32 + lane;
            f.list[pos + __popc(balls[j] & lanemask)] = ((uint32_t)y << 16) | (uint32_t)x;
        }
        pos += __popc(balls[j]);
    }
}

// sizes_by_label[c] = cnt[roots[c]] (ComponentTable::sizes, stage entry)
__global__ void k_sizes_by_label(Frame f, uint32_t* out, int32_t* ids) {
    const uint32_t C = f.sc->n_roots;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        out[c] = f.cnt[f.roots[c]] & ~kRemoved;
        ids[c] = (int32_t)c;
    }
}

// canonical per-pixel labels (-1 on unset pixels), ComponentTable::labels
__global__ void k_labels_out(Frame f, int32_t* out) {
    const long long n = f.N;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        out[i] = f.mref[(size_t)y * f.P + x] ? f.rank[f.par[i]] : -1;
    }
}

// mask.count() into sc->refined_count (stage entry prune_components)
__global__ void k_count_mask(Frame f, const uint8_t* __restrict__ mask) {
    __shared__ unsigned long long red[8];
    unsigned long long n = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < f.N;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        n += mask[(size_t)y * f.P + x] != 0;
    }
    const unsigned long long t = block_sum_u64<256>(n, red);
    if (threadIdx.x == 0 && t) atomicAdd(&f.sc->refined_count, t);
}

// add_border_anchors alone (boundary.cpp:180-195)
__global__ void k_anchor_only(Frame f, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                              int m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < f.N;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / f.W), x = (int)(i - (long long)y * f.W);
        const size_t o = (size_t)y * f.P + x;
        uint8_t v = in[o];
        if ((x == m || x == f.W - 1 - m) && y >= m && y <= f.H - 1 - m) v = 1;
        out[o] = v;
    }
}

}  // namespace

void launch_apply(const Frame& f, bool use_prune, bool anchors, cudaStream_t st) {
    if (f.N == 0) return;
    k_apply<<<f.n_chunks, 256, 0, st>>>(f, use_prune ? 1 : 0, anchors ? 1 : 0);
}

void launch_count_mask(const Frame& f, const uint8_t* mask, cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 8);
    k_count_mask<<<(int)blocks, 256, 0, st>>>(f, mask);
}

void launch_anchor_only(const Frame& f, const uint8_t* in, uint8_t* out, int margin,
                        cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 16);
    k_anchor_only<<<(int)blocks, 256, 0, st>>>(f, in, out, margin);
}

void launch_ccl(const Frame& f, cudaStream_t st) {
    if (f.N == 0) return;
    const dim3 tiles((f.W + CT - 1) / CT, (f.H + CT - 1) / CT);
    k_ccl_local<<<tiles, 256, 0, st>>>(f);
    k_ccl_merge<<<tiles, 128, 0, st>>>(f);
    k_ccl_flatten<<<dim3((f.W + 255) / 256, f.H), 256, 0, st>>>(f);
    k_ccl_roots<<<f.n_chunks, 256, 0, st>>>(f, f.full);
}

void launch_prune(const Frame& f, bool anchors, cudaStream_t st) {
    if (f.N == 0) return;
    k_prune_select<<<1, 1024, 0, st>>>(f);
    k_prune_mark<<<148 * 4, 256, 0, st>>>(f);
    k_apply<<<f.n_chunks, 256, 0, st>>>(f, 1, anchors ? 1 : 0);
}

void launch_component_table(const Frame& f, int32_t* d_labels, uint32_t* d_sizes, int32_t* d_ids,
                            cudaStream_t st) {
    if (f.N == 0) return;
    k_sizes_by_label<<<148 * 2, 256, 0, st>>>(f, d_sizes, d_ids);
    const long long blocks = std::min<long long>((f.N + 255) / 256, 148 * 16);
    k_labels_out<<<(int)blocks, 256, 0, st>>>(f, d_labels);
}

}  // namespace stk
