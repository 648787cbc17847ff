// knn.cu — K2 (exact grid kNN) + K3 (adaptive alpha epilogue) on sm_100a.
//
// Replaces knn_stage / grid_knn (proj/include/aidw/knn.hpp:130-271) and the
// per-query adaptive_alpha chain (adaptive.hpp:20-116).
//
// One thread per query; queries are visited in cell-sorted order (radix
// sort in grid_build.cu) so a warp's 32 queries scan overlapping cell
// blocks and the candidate loads hit L1.  The search is the reference's:
// expansion level = smallest L0 whose clipped (2L0+1)^2 block holds >= k
// points, plus one; scan that block; widen ring by ring until
// kth <= (L*w)^2 (1 - 1e-9) or the block covers the grid.  The k-slot buffer
// is register-resident (RegTopK<KMAX>, KMAX in {4, 16, 32, 64}; a global-
// memory buffer beyond 64) and ordered by the (d2, index) pair, so the value
// list equals the reference's (ties at the kth value are not admitted) and
// the index set is the north-star "ties by index" set.  Every FP64 operation
// uses an explicit round-to-nearest intrinsic and the file is compiled with
// -fmad=false: d2 lists and average distances are bit-identical to the
// reference.
//
// Epilogue per query: r_obs = sum(sqrt(d2), ascending) / k_eff, then
// R = r_obs / r_exp, mu (cosine membership, pi / r_max quirk), alpha
// (triangular levels), plus what the weighting stage needs: d2_min and the
// nearest index (the nearest_value fallback, interpolate.hpp:94-105) and the
// smallest index with d2 <= snap_sq (the snap rule, :127-131).

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "knn.cuh"

namespace aidwb {

namespace {

__device__ __forceinline__ bool pair_less(double da, uint32_t ia, double db, uint32_t ib) {
    return da < db || (da == db && ia < ib);
}

// Register-resident bounded buffer, runtime k <= KMAX.
template <int KMAX>
struct RegTopK {
    double d[KMAX];
    uint32_t id[KMAX];
    int k, filled;
    double kd;
    uint32_t kid;

    __device__ __forceinline__ void init(int kk, double*, uint32_t*) {
        k = kk;
        filled = 0;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            d[j] = __longlong_as_double(0x7FF0000000000000ll);
            id[j] = kNoId;
        }
        kd = d[0];
        kid = kNoId;
    }
    __device__ __forceinline__ bool admits(double cd) const { return cd <= kd; }
    __device__ __forceinline__ void insert(double cd, uint32_t cid) {
        if (!pair_less(cd, cid, kd, kid)) return;
#pragma unroll
        for (int j = KMAX - 1; j >= 1; --j) {
            if (j < k) {
                const bool sp = pair_less(cd, cid, d[j - 1], id[j - 1]);
                const bool sc = pair_less(cd, cid, d[j], id[j]);
                const double nd = sp ? d[j - 1] : (sc ? cd : d[j]);
                const uint32_t ni = sp ? id[j - 1] : (sc ? cid : id[j]);
                d[j] = nd;
                id[j] = ni;
            }
        }
        if (pair_less(cd, cid, d[0], id[0])) {
            d[0] = cd;
            id[0] = cid;
        }
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            if (j == k - 1) {
                kd = d[j];
                kid = id[j];
            }
        }
        filled += filled < k ? 1 : 0;
    }
    __device__ __forceinline__ double get_d(int j) const {
        double r = 0.0;
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
            if (i == j) r = d[i];
        return r;
    }
    __device__ __forceinline__ uint32_t get_id(int j) const {
        uint32_t r = kNoId;
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
            if (i == j) r = id[i];
        return r;
    }
};

// Global-memory bounded buffer for k > 64 (per-query scratch rows).
struct MemTopK {
    double* d;
    uint32_t* id;
    int k, filled;
    double kd;
    uint32_t kid;

    __device__ __forceinline__ void init(int kk, double* dd, uint32_t* ii) {
        d = dd;
        id = ii;
        k = kk;
        filled = 0;
        kd = __longlong_as_double(0x7FF0000000000000ll);
        kid = kNoId;
        for (int j = 0; j < k; ++j) {
            d[j] = kd;
            id[j] = kNoId;
        }
    }
    __device__ __forceinline__ bool admits(double cd) const { return cd <= kd; }
    __device__ void insert(double cd, uint32_t cid) {
        if (!pair_less(cd, cid, kd, kid)) return;
        int pos = k - 1;
        while (pos > 0 && pair_less(cd, cid, d[pos - 1], id[pos - 1])) {
            d[pos] = d[pos - 1];
            id[pos] = id[pos - 1];
            --pos;
        }
        d[pos] = cd;
        id[pos] = cid;
        kd = d[k - 1];
        kid = id[k - 1];
        filled += filled < k ? 1 : 0;
    }
    __device__ __forceinline__ double get_d(int j) const { return d[j]; }
    __device__ __forceinline__ uint32_t get_id(int j) const { return id[j]; }
};

// Offer every point of cell rows [r0, r1] x columns [c0, c1].
template <class TopK>
__device__ __forceinline__ void scan_rect(const KnnArgs& a, TopK& t, double qx, double qy,
                                          int c0, int c1, int r0, int r1, uint32_t& snap,
                                          unsigned long long& scanned) {
    for (int r = r0; r <= r1; ++r) {
        const size_t base = static_cast<size_t>(r) * static_cast<size_t>(a.g.n_col);
        const uint32_t b = __ldg(a.cell_start + base + c0);
        const uint32_t e = __ldg(a.cell_start + base + c1 + 1);
        scanned += e - b;
        for (uint32_t s = b; s < e; ++s) {
            const double cd = dsq_rn(qx, qy, __ldg(a.sorted_x + s), __ldg(a.sorted_y + s));
            if (cd <= a.snap_sq) {
                const uint32_t cid = __ldg(a.sorted_ids + s);
                snap = cid < snap ? cid : snap;
            }
            if (t.admits(cd)) t.insert(cd, __ldg(a.sorted_ids + s));
        }
    }
}

__device__ __forceinline__ size_t rect_count(const KnnArgs& a, int c0, int c1, int r0, int r1) {
    size_t total = 0;
    for (int r = r0; r <= r1; ++r) {
        const size_t base = static_cast<size_t>(r) * static_cast<size_t>(a.g.n_col);
        total += __ldg(a.cell_start + base + c1 + 1) - __ldg(a.cell_start + base + c0);
    }
    return total;
}

__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }

// K3: adaptive alpha (adaptive.hpp:49-87) with reference rounding.
// Returns false (domain error) when mu is outside [0, 1] or NaN.
__device__ __forceinline__ bool alpha_from_robs(const AlphaParams& p, double r_obs,
                                                double& alpha) {
    const double R = __ddiv_rn(r_obs, p.r_exp);
    double mu;
    if (R <= p.r_min) {
        mu = 0.0;
    } else if (R >= p.r_max) {
        mu = 1.0;
    } else {
        const double phase = __dmul_rn(p.pi_over_rmax, __dsub_rn(R, p.r_min));
        mu = __dsub_rn(0.5, __dmul_rn(0.5, cos(phase)));
    }
    if (!(mu >= 0.0 && mu <= 1.0)) return false;
    const double bp[5] = {0.1, 0.3, 0.5, 0.7, 0.9};
    if (mu < bp[0]) {
        alpha = p.lv[0];
        return true;
    }
    if (mu >= bp[4]) {
        alpha = p.lv[4];
        return true;
    }
    int s = 0;
    while (mu >= bp[s + 1]) ++s;
    const double t = __dmul_rn(5.0, __dsub_rn(mu, bp[s]));
    alpha = __dadd_rn(p.lv[s], __dmul_rn(t, __dsub_rn(p.lv[s + 1], p.lv[s])));
    return true;
}

template <class TopK>
__device__ __forceinline__ void finish_query(const KnnArgs& a, TopK& t, size_t pos, uint32_t qi,
                                             uint32_t snap) {
    // ascending sum of square roots (knn.hpp:82-87)
    double sum = 0.0;
    for (int j = 0; j < a.k_eff; ++j) sum = __dadd_rn(sum, __dsqrt_rn(t.get_d(j)));
    const double r_obs = a.k_eff > 0 ? __ddiv_rn(sum, static_cast<double>(a.k_eff)) : 0.0;
    if (a.d2_out) {
        const size_t row = static_cast<size_t>(qi) * static_cast<size_t>(a.k_eff);
        for (int j = 0; j < a.k_eff; ++j) {
            a.d2_out[row + j] = t.get_d(j);
            if (a.id_out) a.id_out[row + j] = t.get_id(j);
        }
    }
    if (a.avg_out) a.avg_out[qi] = r_obs;
    if (a.d2min_s) a.d2min_s[pos] = t.get_d(0);
    if (a.nn_s) a.nn_s[pos] = t.get_id(0);
    if (a.snap_s) a.snap_s[pos] = snap;
    if (a.alpha_s) {
        double alpha = 0.0;
        if (a.compute_alpha) {
            if (!alpha_from_robs(a.ap, r_obs, alpha)) atomicMin(a.fail_alpha, static_cast<long long>(qi));
        } else {
            alpha = a.const_alpha;
        }
        a.alpha_s[pos] = alpha;
    }
}

template <class TopK>
__global__ void __launch_bounds__(128) knn_grid_kernel(KnnArgs a) {
    const size_t pos = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long scanned = 0;
    if (pos < a.n) {
        const uint32_t qi = a.perm[pos];
        const double qx = a.qx[qi], qy = a.qy[qi];
        const uint32_t cell = a.qcell[pos];
        const int n_col = a.g.n_col, n_row = a.g.n_row;
        const int col = static_cast<int>(cell % static_cast<uint32_t>(n_col));
        const int row = static_cast<int>(cell / static_cast<uint32_t>(n_col));

        // expansion level (knn.hpp:130-156)
        int level;
        if (a.m < static_cast<size_t>(a.k)) {
            level = imax(imax(col, n_col - 1 - col), imax(row, n_row - 1 - row));
        } else {
            for (int L0 = 0;; ++L0) {
                const size_t cnt = rect_count(a, imax(0, col - L0), imin(n_col - 1, col + L0),
                                              imax(0, row - L0), imin(n_row - 1, row + L0));
                if (cnt >= static_cast<size_t>(a.k)) {
                    level = L0 + 1;
                    break;
                }
            }
        }

        TopK t;
        t.init(a.k_eff, a.scratch_d + pos * a.k_eff, a.scratch_id + pos * a.k_eff);
        uint32_t snap = kNoId;
        scan_rect(a, t, qx, qy, imax(0, col - level), imin(n_col - 1, col + level),
                  imax(0, row - level), imin(n_row - 1, row + level), snap, scanned);
        // ring widening (knn.hpp:234-247, scan_ring :175-194)
        while (true) {
            const bool covers = col - level <= 0 && row - level <= 0 &&
                                col + level >= n_col - 1 && row + level >= n_row - 1;
            if (covers) break;
            const double reach = __dmul_rn(static_cast<double>(level), a.g.cell_width);
            const double bound = __dmul_rn(__dmul_rn(reach, reach), a.ring_margin);
            if (t.filled == a.k_eff && t.kd <= bound) break;
            ++level;
            const int c0 = imax(0, col - level), c1 = imin(n_col - 1, col + level);
            if (row - level >= 0) scan_rect(a, t, qx, qy, c0, c1, row - level, row - level, snap, scanned);
            if (row + level <= n_row - 1)
                scan_rect(a, t, qx, qy, c0, c1, row + level, row + level, snap, scanned);
            const int pr0 = imax(0, row - (level - 1)), pr1 = imin(n_row - 1, row + (level - 1));
            if (col - level >= 0) scan_rect(a, t, qx, qy, col - level, col - level, pr0, pr1, snap, scanned);
            if (col + level <= n_col - 1)
                scan_rect(a, t, qx, qy, col + level, col + level, pr0, pr1, snap, scanned);
        }
        finish_query(a, t, pos, qi, snap);
    }
    if (a.candidates) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) scanned += __shfl_xor_sync(0xFFFFFFFFu, scanned, o);
        if ((threadIdx.x & 31) == 0 && scanned) atomicAdd(a.candidates, scanned);
    }
}

// Brute-force engine (knn.hpp:100-114): every query scans all m points in
// index order; the data streams through shared memory in 1024-point tiles.
constexpr int kBruteTile = 1024;

template <class TopK>
__global__ void __launch_bounds__(128) knn_brute_kernel(KnnArgs a) {
    __shared__ double sx[kBruteTile], sy[kBruteTile];
    const size_t pos = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = pos < a.n;
    double qx = 0.0, qy = 0.0;
    uint32_t qi = 0;
    if (live) {
        qi = a.perm ? a.perm[pos] : static_cast<uint32_t>(pos);
        qx = a.qx[qi];
        qy = a.qy[qi];
    }
    TopK t;
    t.init(a.k_eff, a.scratch_d + (live ? pos : 0) * a.k_eff,
           a.scratch_id + (live ? pos : 0) * a.k_eff);
    uint32_t snap = kNoId;
    for (size_t base = 0; base < a.m; base += kBruteTile) {
        const int len = static_cast<int>(a.m - base < kBruteTile ? a.m - base : kBruteTile);
        __syncthreads();
        for (int j = threadIdx.x; j < len; j += blockDim.x) {
            sx[j] = a.dx[base + j];
            sy[j] = a.dy[base + j];
        }
        __syncthreads();
        if (live) {
            for (int j = 0; j < len; ++j) {
                const double cd = dsq_rn(qx, qy, sx[j], sy[j]);
                const uint32_t cid = static_cast<uint32_t>(base + j);
                if (cd <= a.snap_sq && cid < snap) snap = cid;
                if (t.admits(cd)) t.insert(cd, cid);
            }
        }
    }
    if (live) finish_query(a, t, pos, qi, snap);
}

#define AIDW_KNN_DISPATCH(KERNEL)                                   \
    do {                                                            \
        const unsigned blocks = ceil_div(a.n, 128);                 \
        if (a.k_eff <= 4) {                                         \
            LAUNCH(KERNEL<RegTopK<4>>, blocks, 128, 0, s, a);       \
        } else if (a.k_eff <= 16) {                                 \
            LAUNCH(KERNEL<RegTopK<16>>, blocks, 128, 0, s, a);      \
        } else if (a.k_eff <= 32) {                                 \
            LAUNCH(KERNEL<RegTopK<32>>, blocks, 128, 0, s, a);      \
        } else if (a.k_eff <= 64) {                                 \
            LAUNCH(KERNEL<RegTopK<64>>, blocks, 128, 0, s, a);      \
        } else {                                                    \
            LAUNCH(KERNEL<MemTopK>, blocks, 128, 0, s, a);          \
        }                                                           \
    } while (0)

}  // namespace

void run_knn_grid(KnnArgs a, cudaStream_t s) {
    if (a.n == 0) return;
    DBuf<double> sd;
    DBuf<uint32_t> si;
    if (a.k_eff > 64) {
        sd.alloc(a.n * static_cast<size_t>(a.k_eff), s);
        si.alloc(a.n * static_cast<size_t>(a.k_eff), s);
        a.scratch_d = sd.get();
        a.scratch_id = si.get();
    }
    AIDW_KNN_DISPATCH(knn_grid_kernel);
}

void run_knn_brute(KnnArgs a, cudaStream_t s) {
    if (a.n == 0) return;
    DBuf<double> sd;
    DBuf<uint32_t> si;
    if (a.k_eff > 64) {
        sd.alloc(a.n * static_cast<size_t>(a.k_eff), s);
        si.alloc(a.n * static_cast<size_t>(a.k_eff), s);
        a.scratch_d = sd.get();
        a.scratch_id = si.get();
    }
    AIDW_KNN_DISPATCH(knn_brute_kernel);
}

namespace {
// K3 alone: alpha from caller-supplied r_obs (aidw_predict_all drop-in path).
__global__ void alpha_kernel(const double* __restrict__ r_obs, size_t n, AlphaParams p,
                             double* __restrict__ alpha, long long* __restrict__ fail) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a = 0.0;
    if (!alpha_from_robs(p, r_obs[i], a)) atomicMin(fail, static_cast<long long>(i));
    alpha[i] = a;
}
}  // namespace

void run_alpha(const double* d_robs, size_t n, const AlphaParams& p, double* d_alpha,
               long long* d_fail, cudaStream_t s) {
    if (n == 0) return;
    LAUNCH(alpha_kernel, ceil_div(n, kThreads), kThreads, 0, s, d_robs, n, p, d_alpha, d_fail);
}

}  // namespace aidwb
