// K2 kmeans_warp -- Lloyd K-Means over the 256 histogram bins, one warp,
// exact FP64 (reference: segmentation.cpp:49-144, caller pipeline.cpp:72-85).
//
// Lane l owns bins 8l..8l+7.  Every floating-point step uses the _rn
// intrinsics in the reference's operation order so no DFMA contraction can
// change a center: init lo + (hi-lo)*(j/(k-1.0)); |v - c| distances with
// strict '<' (ties to the lowest index); center = double(sum)/double(weight)
// from exact u64 sums; stop when max movement < tol or after max_iter.  The
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
__global__ void __launch_bounds__(32) k_kmeans(Frame f, int k_fixed, int max_iter, double tol) {
    __shared__ double c[256];
    __shared__ unsigned long long wsum[256], vsum[256];
    DevScalars* sc = f.sc;
    const int lane = threadIdx.x;
    unsigned long long cnt[8];
    int occ = 0, lo = 256, hi = -1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int v = lane * 8 + i;
        cnt[i] = sc->hist[v];
        if (cnt[i]) {
            ++occ;
            lo = min(lo, v);
            hi = max(hi, v);
        }
    }
    occ = __reduce_add_sync(0xffffffffu, occ);
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    int k;
    if (k_fixed > 0) {
        k = k_fixed;
    } else {
        k = min(f.kcfg, occ);
    }
    if (occ == 0 || k < 1 || k > occ) {
        if (lane == 0) {
            sc->kerr = occ == 0 ? 1 : (k < 1 ? 3 : 2);
            sc->k = 0;
        }
        return;
    }
    // init (segmentation.cpp:96-102)
    for (int j = lane; j < k; j += 32) {
        if (k == 1)
            c[j] = __ddiv_rn((double)(lo + hi), 2.0);
        else
            c[j] = __dadd_rn((double)lo, __dmul_rn((double)(hi - lo),
                                                   __ddiv_rn((double)j, __dsub_rn((double)k, 1.0))));
    }
    __syncwarp();
    int iters = 0;
    for (int it = 1; it <= max_iter; ++it) {
        for (int j = lane; j < k; j += 32) wsum[j] = vsum[j] = 0ull;
        __syncwarp();
        // assignment of all 256 bins; sums over occupied bins (:104-120)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (!cnt[i]) continue;
            const int v = lane * 8 + i;
            const int a = nearest(c, k, (double)v);
            atomicAdd(&wsum[a], cnt[i]);
            atomicAdd(&vsum[a], cnt[i] * (unsigned long long)v);
        }
        __syncwarp();
        // update (:122-135); movement = max |updated - old| over non-empty clusters
        double move = 0.0;
        for (int j = lane; j < k; j += 32) {
            if (wsum[j] == 0ull) continue;
            const double upd = __ddiv_rn(__ull2double_rn(vsum[j]), __ull2double_rn(wsum[j]));
            const double m = fabs(__dsub_rn(upd, c[j]));
            if (move < m) move = m;
            c[j] = upd;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) move = fmax(move, __shfl_xor_sync(0xffffffffu, move, o));
        __syncwarp();
        iters = it;
        if (move < tol) break;
    }
    // final table against final centers (:139-142)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int v = lane * 8 + i;
        const int a = nearest(c, k, (double)v);
        sc->assign16[v] = (unsigned short)a;
        sc->lut[v] = (unsigned char)a;
    }
    for (int j = lane; j < 256; j += 32) sc->centers[j] = j < k ? c[j] : 0.0;
    if (lane == 0) {
        sc->k = k;
        sc->iters = iters;
        sc->kerr = 0;
    }
}

}  // namespace

void launch_kmeans(const Frame& f, int k_fixed, int max_iter, double tol, cudaStream_t st) {
    k_kmeans<<<1, 32, 0, st>>>(f, k_fixed, max_iter, tol);
}

}  // namespace stk
