// K4 -- connected components, prune, anchors and boundary-pixel compaction,
// all on the device with no host round trip (reference: boundary.cpp:87-195,
// pipeline.cpp:92-94).
//
//   K4a ccl_local    one warp per 32x32 tile: lane = row, the row is a 32-bit
//                    mask, runs (maximal horizontal segments) are the
//                    union-find nodes; runs of adjacent rows that touch
//                    (8-connectivity) are united with atomicMin in shared
//                    memory, paths compressed, and run lengths summed into
//                    local component sizes.  Every pixel's parent becomes its
//                    local root (min raster index of the local component); the
//                    local roots go to a list with their sizes.
//   K4b ccl_merge    tile-border pixels unite across tiles in global memory
//                    (lock-free atomicMin union on raster indices).
//   K4c ccl_compress one thread per local root: find + path compression to the
//                    global root (= min raster index of the component), local
//                    size added to the global size.  A pixel's root is then
//                    par[par[i]].
//   K4d ccl_roots    ordered compaction of global roots (single-pass decoupled
//                    look-back): canonical label = rank of the root in raster
//                    order, exactly the reference's discovery order; size
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

constexpr int CT = 32;          // CCL tile side
constexpr int kLocalWarps = 4;  // tiles per K4a CTA

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

__device__ __forceinline__ uint32_t upto_mask(int j) {  // bits 0..j
    return j >= 31 ? 0xffffffffu : ((2u << j) - 1u);
}

__device__ __forceinline__ int run_len(uint32_t m, int a) {  // set bits from a upward
    const uint32_t inv = ~(m >> a);
    return inv ? __ffs(inv) - 1 : 32 - a;
}

// 32 mask bytes (0 / nonzero) -> 32-bit row mask
__device__ __forceinline__ uint32_t bytes_to_bits(uint4 a, uint4 b) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t v = __vcmpne4(w[i], 0u) & 0x01010101u;
        m |= ((v * 0x01020408u) >> 24) << (4 * i);
    }
    return m;
}

// ----------------------------------------------------------------- K4a ----
__global__ void __launch_bounds__(32 * kLocalWarps) k_ccl_local(Frame f) {
    __shared__ int sp[kLocalWarps][CT * CT];
    __shared__ int ssz[kLocalWarps][CT * CT];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {   // zero the size-histogram bins the prune will use (0..B+1)
        const unsigned long long B = budget_of(f);
        const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
        const long long stride = (long long)gridDim.x * blockDim.x;
        for (long long s = gt; s <= (long long)B + 1; s += stride) f.szhist[s] = 0;
        if (gt == 0) f.sc->budget = B;
    }
    const int TXc = (f.W + CT - 1) / CT, TYc = (f.H + CT - 1) / CT;
    const int tile = blockIdx.x * kLocalWarps + wid;
    if (tile >= TXc * TYc) return;
    const int x0 = (tile % TXc) * CT, y0 = (tile / TXc) * CT;
    int* p = sp[wid];
    int* sz = ssz[wid];
    uint32_t m = 0;
    if (y0 + lane < f.H) {
        const uint4* row = reinterpret_cast<const uint4*>(f.mref + (size_t)(y0 + lane) * f.P + x0);
        m = bytes_to_bits(row[0], row[1]);
        if (f.W - x0 < 32) m &= (1u << (f.W - x0)) - 1u;
    }
    const uint32_t s = m & ~(m << 1);  // run starts
    for (uint32_t t = s; t; t &= t - 1) {
        const int node = lane * 32 + __ffs(t) - 1;
        p[node] = node;
        sz[node] = 0;
    }
    __syncwarp();
    uint32_t mu = __shfl_up_sync(0xffffffffu, m, 1), su = __shfl_up_sync(0xffffffffu, s, 1);
    if (lane == 0) mu = su = 0;
    for (uint32_t t = s; t; t &= t - 1) {
        const int a = __ffs(t) - 1;
        const int b = a + run_len(m, a) - 1;
        const int lo = a > 0 ? a - 1 : 0, hi = b < 31 ? b + 1 : 31;
        uint32_t T = mu & upto_mask(hi) & ~((1u << lo) - 1u);
        while (T) {
            const int j = __ffs(T) - 1;
            const int sa = 31 - __clz(su & upto_mask(j));
            sunite(p, lane * 32 + a, (lane - 1) * 32 + sa);
            const int e = sa + run_len(mu, sa) - 1;
            T &= e >= 31 ? 0u : ~upto_mask(e);
        }
    }
    __syncwarp();
    int nroots = 0;
    for (uint32_t t = s; t; t &= t - 1) {
        const int a = __ffs(t) - 1, node = lane * 32 + a;
        const int r = sfind(p, node);
        p[node] = r;
        atomicAdd(&sz[r], run_len(m, a));
        nroots += r == node;
    }
    __syncwarp();
    // local roots -> list (unordered), zero their global size
    int incl = nroots;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    unsigned base = 0;
    if (lane == 31 && incl) base = atomicAdd(&f.sc->n_lroots, (unsigned)incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    unsigned pos = base + incl - nroots;
    uint32_t* lr_idx = f.list;
    uint32_t* lr_size = reinterpret_cast<uint32_t*>(f.rank);
    for (uint32_t t = s; t; t &= t - 1) {
        const int node = lane * 32 + __ffs(t) - 1;
        if (p[node] == node) {
            const int g = (y0 + lane) * f.W + x0 + (node & 31);
            lr_idx[pos] = (uint32_t)g;
            lr_size[pos] = (uint32_t)sz[node];
            f.cnt[g] = 0;
            ++pos;
        }
    }
    // every pixel -> its local root (coalesced: the warp walks the rows)
    for (int rr = 0; rr < CT; ++rr) {
        const uint32_t mr = __shfl_sync(0xffffffffu, m, rr), sr = __shfl_sync(0xffffffffu, s, rr);
        if ((mr >> lane) & 1u) {
            const int st = 31 - __clz(sr & upto_mask(lane));
            const int root = p[rr * 32 + st];
            f.par[(y0 + rr) * f.W + x0 + lane] = (y0 + (root >> 5)) * f.W + x0 + (root & 31);
        }
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
__global__ void __launch_bounds__(256) k_ccl_compress(Frame f) {
    const unsigned n = f.sc->n_lroots;
    const uint32_t* lr_idx = f.list;
    const uint32_t* lr_size = reinterpret_cast<const uint32_t*>(f.rank);
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int lr = (int)lr_idx[i];
        const int r = gfind(f.par, lr);
        int x = lr;
        while (true) {  // path compression (all writers store the same root)
            const int nx = __ldcg(f.par + x);
            if (nx == x || nx == r) break;
            f.par[x] = r;
            x = nx;
        }
        if (x != r) f.par[x] = r;
        atomicAdd(f.cnt + r, lr_size[i]);
    }
}

// ----------------------------------------------------------------- K4d ----
// Chunk = 32 row-tiles; warp w owns tiles 4w..4w+3 of the chunk (128 pixels
// of one row each, 4 per lane at x = seg*128 + j*32 + lane) so ballots come
// out in raster order.
__global__ void __launch_bounds__(256) k_ccl_roots(Frame f, int write_rank) {
    __shared__ uint32_t s_chunk, s_excl;
    __shared__ uint32_t wcount[8];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* status = f.lb + LB_ROOTS * f.lb_stride;
    if (threadIdx.x == 0) s_chunk = atomicAdd(&f.sc->ctr[LB_ROOTS], 1u);
    __syncthreads();
    const int c = s_chunk;
    const int t0 = c * kTilesPerChunk + wid * kTilesPerWarp;
    uint32_t balls[kTilesPerWarp][4];
    uint32_t wc = 0;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        const int y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = seg * kRowTile + j * 32 + lane;
            bool isroot = false;
            if (t < f.n_tiles && x < f.W && f.mref[(size_t)y * f.P + x]) {
                const int g = y * f.W + x;
                isroot = __ldg(f.par + g) == g;
            }
            balls[k][j] = __ballot_sync(0xffffffffu, isroot);
            wc += __popc(balls[k][j]);
        }
    }
    if (lane == 0) wcount[wid] = wc;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < 8 ? wcount[lane] : 0u;
        const uint32_t agg = __reduce_add_sync(0xffffffffu, v);
        const uint32_t excl = lb_exclusive_warp(status, c, agg);
        if (lane == 0) {
            s_excl = excl;
            if (c == f.n_chunks - 1) f.sc->n_roots = excl + agg;
        }
    }
    __syncthreads();
    uint32_t pos = s_excl;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    const unsigned long long B = f.sc->budget;
    const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        const int y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (balls[k][j] >> lane & 1u) {
                const int g = y * f.W + seg * kRowTile + j * 32 + lane;
                const uint32_t p = pos + __popc(balls[k][j] & lanemask);
                f.roots[p] = g;
                if (write_rank) f.rank[g] = (int)p;
                const uint32_t sz = f.cnt[g];
                if (sz <= B + 1) atomicAdd(f.szhist + sz, 1u);
            }
            pos += __popc(balls[k][j]);
        }
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
            if (wid == 0) {
                const uint32_t agg = __reduce_add_sync(0xffffffffu, lane < 8 ? wcount[lane] : 0u);
                const uint32_t excl = lb_exclusive_warp(status, (int)c, agg);
                if (lane == 0) s_excl = excl;
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
    const int t0 = c * kTilesPerChunk + wid * kTilesPerWarp;
    const int m = f.hw, W = f.W, H = f.H;
    uint32_t balls[kTilesPerWarp][4];
    uint32_t wc = 0, kept = 0;
    unsigned long long ops = 0;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        const bool tv = t < f.n_tiles;
        const int y = t / f.TX, seg = t % f.TX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = seg * kRowTile + j * 32 + lane;
            bool keep = false, anc = false;
            if (tv && x < W) {
                const size_t po = (size_t)y * f.P + x;
                const int g = y * W + x;
                if (f.mref[po]) {
                    if (use_prune) {
                        const int r = __ldg(f.par + __ldg(f.par + g));
                        keep = !(__ldg(f.cnt + r) & kRemoved);
                    } else {
                        keep = true;
                    }
                }
                anc = keep;
                if (anchors && (x == m || x == W - 1 - m) && y >= m && y <= H - 1 - m) anc = true;
                if (f.mprn) f.mprn[po] = keep;
                if (f.manc) f.manc[po] = anc;
                f.sparse[g] = -1;
            }
            kept += keep;
            const bool matchable = anc && y >= m && y < H - m && x >= m && x < W - m;
            balls[k][j] = __ballot_sync(0xffffffffu, matchable);
            wc += __popc(balls[k][j]);
            if (matchable) ops += (unsigned long long)(min(f.D, x - m) + 1);
            if (tv && lane == 0) f.mbits[(size_t)y * f.bits_words + seg * 4 + j] = balls[k][j];
        }
    }
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
    if (wid == 0) {
        const uint32_t agg = __reduce_add_sync(0xffffffffu, lane < 8 ? wcount[lane] : 0u);
        const uint32_t excl = lb_exclusive_warp(status, c, agg);
        if (lane == 0) {
            s_excl = excl;
            unsigned long long ka = 0, oa = 0;
            for (int i = 0; i < 8; ++i) {
                ka += red[i];
                oa += red2[i];
            }
            if (ka) atomicAdd(&f.sc->pruned_count, ka);
            if (oa) atomicAdd(&f.sc->sad_ops, oa * (unsigned long long)(f.window * f.window));
            if (c == f.n_chunks - 1) {
                f.sc->n_list = excl + agg;
                f.sc->matched = excl + agg;
                f.tile_off[f.n_tiles] = excl + agg;
            }
        }
    }
    __syncthreads();
    uint32_t pos = s_excl;
    for (int i = 0; i < wid; ++i) pos += wcount[i];
    const uint32_t lanemask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kTilesPerWarp; ++k) {
        const int t = t0 + k;
        if (t >= f.n_tiles) break;
        const int y = t / f.TX, seg = t % f.TX;
        if (lane == 0) f.tile_off[t] = pos;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (balls[k][j] >> lane & 1u) {
                const int x = seg * kRowTile + j * 32 + lane;
                f.list[pos + __popc(balls[k][j] & lanemask)] = ((uint32_t)y << 16) | (uint32_t)x;
            }
            pos += __popc(balls[k][j]);
        }
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
        out[i] = f.mref[(size_t)y * f.P + x] ? f.rank[f.par[f.par[i]]] : -1;
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
    const long long blocks = std::min<long long>((f.N + 255) / 256, f.sms * 8);
    k_count_mask<<<(int)blocks, 256, 0, st>>>(f, mask);
}

void launch_anchor_only(const Frame& f, const uint8_t* in, uint8_t* out, int margin,
                        cudaStream_t st) {
    if (f.N == 0) return;
    const long long blocks = std::min<long long>((f.N + 255) / 256, f.sms * 16);
    k_anchor_only<<<(int)blocks, 256, 0, st>>>(f, in, out, margin);
}

void launch_ccl(const Frame& f, cudaStream_t st) {
    if (f.N == 0) return;
    const dim3 tiles((f.W + CT - 1) / CT, (f.H + CT - 1) / CT);
    const int ntiles = tiles.x * tiles.y;
    k_ccl_local<<<(ntiles + kLocalWarps - 1) / kLocalWarps, 32 * kLocalWarps, 0, st>>>(f);
    k_ccl_merge<<<tiles, 128, 0, st>>>(f);
    k_ccl_compress<<<f.sms * 8, 256, 0, st>>>(f);
    k_ccl_roots<<<f.n_chunks, 256, 0, st>>>(f, f.full);
}

void launch_ccl_compress(const Frame& f, cudaStream_t st) {
    if (f.N == 0) return;
    k_ccl_compress<<<f.sms * 8, 256, 0, st>>>(f);
}

void launch_prune_select(const Frame& f, cudaStream_t st) {
    if (f.N == 0) return;
    k_prune_select<<<1, 1024, 0, st>>>(f);
}

void launch_prune(const Frame& f, bool anchors, cudaStream_t st) {
    if (f.N == 0) return;
    k_prune_select<<<1, 1024, 0, st>>>(f);
    k_prune_mark<<<f.sms * 4, 256, 0, st>>>(f);
    k_apply<<<f.n_chunks, 256, 0, st>>>(f, 1, anchors ? 1 : 0);
}

void launch_component_table(const Frame& f, int32_t* d_labels, uint32_t* d_sizes, int32_t* d_ids,
                            cudaStream_t st) {
    if (f.N == 0) return;
    k_sizes_by_label<<<f.sms * 2, 256, 0, st>>>(f, d_sizes, d_ids);
    const long long blocks = std::min<long long>((f.N + 255) / 256, f.sms * 16);
    k_labels_out<<<(int)blocks, 256, 0, st>>>(f, d_labels);
}

}  // namespace stk
