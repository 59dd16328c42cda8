// K2 kmeans_hist -- Lloyd K-Means over the 256 histogram bins, one CTA of 256
// threads (one bin each), exact FP64 (reference: segmentation.cpp:49-144,
// caller pipeline.cpp:72-85).
//
// Every floating-point step uses the _rn intrinsics in the reference's
// operation order so no DFMA contraction can change a center: init
// lo + (hi-lo)*(j/(k-1.0)); |v - c| distances with strict '<' (ties to the
// lowest index); center = double(sum)/double(weight) from exact u64 sums;
// stop when max movement < tol or after max_iter.  Per-cluster sums: lanes of
// a warp holding the same cluster are grouped with __match_any_sync and the
// group leader adds the group's sums (one shared u64 atomic per group).  The
// effective k = min(cfg.k, occupied bins) is decided on the device, so the
// frame never syncs with the host.
#include "stk_device.cuh"

namespace stk {

namespace {

__device__ __forceinline__ int nearest(const double* c, int k, double v) {
    int best = 0;
    double bd = fabs(__dsub_rn(v, c[0]));
    for (int j = 1; j < k; ++j) {
        const double d = fabs(__dsub_rn(v, c[j]));
        if (d < bd) {
            bd = d;
            best = j;
        }
    }
    return best;
}

// k_fixed > 0: use exactly that k (stage entry kmeans_histogram, which must
// reject k > occupied); k_fixed <= 0: k = min(f.kcfg, occupied) (pipeline).
__global__ void __launch_bounds__(256) k_kmeans(Frame f, int k_fixed, int max_iter, double tol) {
    __shared__ double c[256];
    __shared__ unsigned long long wsum[256], vsum[256];
    __shared__ unsigned long long gw[256], gv[256];  // per-lane staging for group sums
    __shared__ double wmove[8];
    __shared__ int s_lo[8], s_hi[8];
    DevScalars* sc = f.sc;
    const int v = threadIdx.x, lane = v & 31, wid = v >> 5;
    const unsigned long long cnt = sc->hist[v];
    const int occ = __syncthreads_count(cnt != 0);
    int lo = __reduce_min_sync(0xffffffffu, cnt ? v : 256);
    int hi = __reduce_max_sync(0xffffffffu, cnt ? v : -1);
    if (lane == 0) {
        s_lo[wid] = lo;
        s_hi[wid] = hi;
    }
    __syncthreads();
    lo = 256;
    hi = -1;
    for (int i = 0; i < 8; ++i) {
        lo = min(lo, s_lo[i]);
        hi = max(hi, s_hi[i]);
    }
    const int k = k_fixed > 0 ? k_fixed : min(f.kcfg, occ);
    if (occ == 0 || k < 1 || k > occ) {
        if (v == 0) {
            sc->kerr = occ == 0 ? 1 : (k < 1 ? 3 : 2);
            sc->k = 0;
        }
        return;
    }
    // init (segmentation.cpp:96-102)
    if (v < k) {
        if (k == 1)
            c[v] = __ddiv_rn((double)(lo + hi), 2.0);
        else
            c[v] = __dadd_rn((double)lo, __dmul_rn((double)(hi - lo),
                                                   __ddiv_rn((double)v, __dsub_rn((double)k, 1.0))));
    }
    __syncthreads();
    int iters = 0;
    for (int it = 1; it <= max_iter; ++it) {
        wsum[v] = vsum[v] = 0ull;
        // assignment of all bins; sums over occupied bins (:104-120)
        const int a = nearest(c, k, (double)v);
        gw[v] = cnt;
        gv[v] = cnt * (unsigned long long)v;
        __syncthreads();
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        if ((__ffs(peers) - 1) == lane) {
            unsigned long long sw = 0, sv = 0;
            for (unsigned m = peers; m; m &= m - 1) {
                const int l = (wid << 5) + __ffs(m) - 1;
                sw += gw[l];
                sv += gv[l];
            }
            if (sw) {
                atomicAdd(&wsum[a], sw);
                atomicAdd(&vsum[a], sv);
            }
        }
        __syncthreads();
        // update (:122-135); movement = max |updated - old| over non-empty clusters
        double move = 0.0;
        if (v < k && wsum[v] != 0ull) {
            const double upd = __ddiv_rn(__ull2double_rn(vsum[v]), __ull2double_rn(wsum[v]));
            move = fabs(__dsub_rn(upd, c[v]));
            c[v] = upd;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) move = fmax(move, __shfl_xor_sync(0xffffffffu, move, o));
        if (lane == 0) wmove[wid] = move;
        __syncthreads();
        move = wmove[0];
        for (int i = 1; i < 8; ++i) move = fmax(move, wmove[i]);
        iters = it;
        if (move < tol) break;
    }
    // final table against final centers (:139-142)
    const int a = nearest(c, k, (double)v);
    sc->assign16[v] = (unsigned short)a;
    sc->lut[v] = (unsigned char)a;
    sc->centers[v] = v < k ? c[v] : 0.0;
    if (v == 0) {
        sc->k = k;
        sc->iters = iters;
        sc->kerr = 0;
    }
}

// One-warp variant for k <= 32 (the pipeline's K): lane l owns bins
// 8l..8l+7, no block barriers.  Every 1-D nearest-center cell is an interval
// of bins (strict '<', ties to the lowest index, any center order), so each
// cluster's exact u64 sums are differences of prefix sums of (count,
// count * v) built once; the centers, movements and iteration count follow the
// reference exactly as in k_kmeans.
__global__ void __launch_bounds__(32) k_kmeans_warp(Frame f, int k_fixed, int max_iter, double tol) {
    __shared__ double c[32];
    __shared__ unsigned long long pw[257], pv[257];  // exclusive prefix sums
    __shared__ int first[32], last[32];
    DevScalars* sc = f.sc;
    const int lane = threadIdx.x;
    unsigned long long cnt[8];
    int nocc = 0, lo = 256, hi = -1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int v = 8 * lane + i;
        cnt[i] = sc->hist[v];
        if (cnt[i]) {
            ++nocc;
            lo = min(lo, v);
            hi = max(hi, v);
        }
    }
    const int occ = __reduce_add_sync(0xffffffffu, nocc);
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    const int k = k_fixed > 0 ? k_fixed : min(f.kcfg, occ);
    if (occ == 0 || k < 1 || k > occ) {
        if (lane == 0) {
            sc->kerr = occ == 0 ? 1 : (k < 1 ? 3 : 2);
            sc->k = 0;
        }
        return;
    }
    {   // prefix sums
        unsigned long long sw = 0, sv = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            sw += cnt[i];
            sv += cnt[i] * (unsigned long long)(8 * lane + i);
        }
        unsigned long long iw = sw, iv = sv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long a = __shfl_up_sync(0xffffffffu, iw, o);
            const unsigned long long b = __shfl_up_sync(0xffffffffu, iv, o);
            if (lane >= o) iw += a, iv += b;
        }
        unsigned long long w0 = iw - sw, v0 = iv - sv;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            pw[8 * lane + i] = w0;
            pv[8 * lane + i] = v0;
            w0 += cnt[i];
            v0 += cnt[i] * (unsigned long long)(8 * lane + i);
        }
        if (lane == 31) pw[256] = w0, pv[256] = v0;
    }
    if (lane < k) {
        if (k == 1)
            c[lane] = __ddiv_rn((double)(lo + hi), 2.0);
        else
            c[lane] = __dadd_rn((double)lo, __dmul_rn((double)(hi - lo),
                                                      __ddiv_rn((double)lane, __dsub_rn((double)k, 1.0))));
    }
    __syncwarp();
    int iters = 0;
    int a[8];
    for (int it = 1; it <= max_iter; ++it) {
        if (lane < k) first[lane] = -1;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = nearest(c, k, (double)(8 * lane + i));
        // interval starts / ends of the cells
        const int aprev = __shfl_up_sync(0xffffffffu, a[7], 1);
        const int anext = __shfl_down_sync(0xffffffffu, a[0], 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int v = 8 * lane + i;
            const int pa = i > 0 ? a[i - 1] : (lane > 0 ? aprev : -1);
            const int na = i < 7 ? a[i + 1] : (lane < 31 ? anext : -1);
            if (a[i] != pa) first[a[i]] = v;
            if (a[i] != na) last[a[i]] = v;
        }
        __syncwarp();
        double move = 0.0;
        if (lane < k && first[lane] >= 0) {
            const unsigned long long w = pw[last[lane] + 1] - pw[first[lane]];
            if (w != 0ull) {
                const unsigned long long vs = pv[last[lane] + 1] - pv[first[lane]];
                const double upd = __ddiv_rn(__ull2double_rn(vs), __ull2double_rn(w));
                move = fabs(__dsub_rn(upd, c[lane]));
                c[lane] = upd;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) move = fmax(move, __shfl_xor_sync(0xffffffffu, move, o));
        __syncwarp();
        iters = it;
        if (move < tol) break;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int v = 8 * lane + i;
        const int aa = nearest(c, k, (double)v);
        sc->assign16[v] = (unsigned short)aa;
        sc->lut[v] = (unsigned char)aa;
        sc->centers[v] = v < k ? c[v] : 0.0;
    }
    if (lane == 0) {
        sc->k = k;
        sc->iters = iters;
        sc->kerr = 0;
    }
}

}  // namespace

void launch_kmeans(const Frame& f, int k_fixed, int max_iter, double tol, cudaStream_t st) {
    const int kmax = k_fixed > 0 ? k_fixed : f.kcfg;
    if (kmax <= 32) k_kmeans_warp<<<1, 32, 0, st>>>(f, k_fixed, max_iter, tol);
    else k_kmeans<<<1, 256, 0, st>>>(f, k_fixed, max_iter, tol);
}

}  // namespace stk
