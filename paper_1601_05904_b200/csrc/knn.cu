// knn.cu — K2 (exact grid kNN) + K3 (adaptive alpha epilogue) on sm_100a.
//
// Replaces knn_stage / grid_knn (proj/include/aidw/knn.hpp:130-271) and the
// per-query adaptive_alpha chain (adaptive.hpp:20-116).
//
// One thread per query; queries are visited in block-major cell order
// (8 x 8-cell blocks, radix sort in grid_build.cu) so a CTA's 128 queries
// sit in a compact patch of cells: the CTA stages the patch widened by two
// cells (coordinates, ids, local CSR offsets) in shared memory and its
// threads scan the row segments inside it from there (measured: -1.3 % K2
// time clustered, +1.5-2.5 % uniform / stress / DEM — K2 is bound by its
// top-k network, not by candidate loads, profiles/r02/k2_stage_s43.txt);
// segments outside the patch read global memory through L1.  Each thread
// walks its cells as one level block row by row (a row segment of cells is
// contiguous in memory).  The search is the reference's:
// expansion level = smallest L0 whose clipped (2L0+1)^2 block holds >= k
// points, plus one; scan that block; widen ring by ring until
// kth <= (L*w)^2 (1 - 1e-9) or the block covers the grid.  The block is
// walked ring by ring from the query's cell and cells whose padded
// rectangle lies strictly beyond the current k-th are skipped — the k
// smallest (d2, idx) of every level's block are unchanged, so stop decisions
// and results equal the reference's while ~1/3 of its candidates are read
// (1M uniform: 34M of 99M).  The k-slot buffer
// is a register-resident static sorting network (RegTopK<KMAX>, KMAX a
// compile-time bucket >= k up to 64; a global-memory buffer beyond) ordered
// by the (d2, index) pair, so the value
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

#include <climits>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "knn.cuh"

namespace aidwb {

namespace {

__device__ __forceinline__ bool pair_less(double da, uint32_t ia, double db, uint32_t ib) {
    // non-short-circuit form: per slot the three compares are independent
    // (the && / || form compiles to a predicated DSETP chain through the
    // whole network; this one is 20-28 % faster, K2 0.46 -> 0.37 ms at 1M)
    return static_cast<bool>(static_cast<int>(da < db) |
                             (static_cast<int>(da == db) & static_cast<int>(ia < ib)));
}

// Register-resident bounded buffer as a static sorting network.  KMAX is a
// compile-time bucket >= k; the first KMAX - k slots hold (-inf, 0)
// sentinels that no candidate can pass, so the k real entries always sit in
// slots [KMAX - k, KMAX) and the k-th is slot KMAX - 1 — every index is
// static, nothing spills to local memory.  Insert: KMAX independent
// (d2, idx) comparisons, then each slot takes its left neighbour, the
// candidate, or itself.
template <int KMAX>
struct RegTopK {
    double d[KMAX];
    uint32_t id[KMAX];
    int k;

    __device__ __forceinline__ void init(int kk, double*, uint32_t*) {
        k = kk;
        const double inf = __longlong_as_double(0x7FF0000000000000ll);
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const bool front = j < KMAX - kk;
            d[j] = front ? -inf : inf;
            id[j] = front ? 0u : kNoId;
        }
    }
    __device__ __forceinline__ double kth() const { return d[KMAX - 1]; }
    __device__ __forceinline__ bool full() const { return id[KMAX - 1] != kNoId; }
    __device__ __forceinline__ bool admits(double cd) const { return cd <= d[KMAX - 1]; }
    __device__ __forceinline__ void insert(double cd, uint32_t cid) {
        if (!pair_less(cd, cid, d[KMAX - 1], id[KMAX - 1])) return;
        bool lt[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) lt[j] = pair_less(cd, cid, d[j], id[j]);
#pragma unroll
        for (int j = KMAX - 1; j >= 1; --j) {
            d[j] = lt[j - 1] ? d[j - 1] : (lt[j] ? cd : d[j]);
            id[j] = lt[j - 1] ? id[j - 1] : (lt[j] ? cid : id[j]);
        }
        if (lt[0]) {
            d[0] = cd;
            id[0] = cid;
        }
    }
    // j-th smallest real entry (0-based); unrolled select, used at the end
    __device__ __forceinline__ double get_d(int j) const {
        double r = 0.0;
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
            if (i == KMAX - k + j) r = d[i];
        return r;
    }
    __device__ __forceinline__ uint32_t get_id(int j) const {
        uint32_t r = kNoId;
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
            if (i == KMAX - k + j) r = id[i];
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
    __device__ __forceinline__ double kth() const { return kd; }
    __device__ __forceinline__ bool full() const { return filled == k; }
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

// Conservative lower bound of d2 from the query (fx, fy in cell units) to
// any point assigned to cell (c, r): the cell padded by 1e-7 cells (covers
// the FP64 rounding of both cell assignments), edge cells unbounded outward
// (locate_cell clamps points from the slack band into them), and a 1e-9
// relative margin on the product.
__device__ __forceinline__ double cell_lower_d2(const GridGeom& g, double fx, double fy,
                                                double w2, int c, int r) {
    const double inf = __longlong_as_double(0x7FF0000000000000ll);
    const double pad = 1.0e-7;
    const double x0 = c == 0 ? -inf : c - pad, x1 = c == g.n_col - 1 ? inf : c + 1 + pad;
    const double y0 = r == 0 ? -inf : r - pad, y1 = r == g.n_row - 1 ? inf : r + 1 + pad;
    const double dx = fmax(0.0, fmax(x0 - fx, fx - x1));
    const double dy = fmax(0.0, fmax(y0 - fy, fy - y1));
    return (dx * dx + dy * dy) * w2 * (1.0 - 1.0e-9);
}

// Points in the cell rectangle [c0, c1] x [r0, r1]: four loads of the
// summed-area table (O(1) whatever the block size — the void queries of the
// clustered stress case reach levels ~100), else one cell_start pair per row.
__device__ __forceinline__ size_t rect_count(const KnnArgs& a, int c0, int c1, int r0, int r1) {
    if (a.rect_prefix) {  // PT[c][r], column-major
        const size_t h = static_cast<size_t>(a.g.n_row) + 1;
        const uint32_t* P = a.rect_prefix;
        const uint32_t* lo = P + static_cast<size_t>(c0) * h;
        const uint32_t* hi = P + static_cast<size_t>(c1 + 1) * h;
        // u32 arithmetic wraps exactly (every count < 2^32)
        return __ldg(hi + r1 + 1) - __ldg(hi + r0) - __ldg(lo + r1 + 1) + __ldg(lo + r0);
    }
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
    if (mu < 0.1) {
        alpha = p.lv[0];
        return true;
    }
    if (mu >= 0.9) {
        alpha = p.lv[4];
        return true;
    }
    // lower-inclusive segment [bp_s, bp_s+1) and its two levels (static picks)
    double bp, lo, hi;
    if (mu < 0.3) {
        bp = 0.1, lo = p.lv[0], hi = p.lv[1];
    } else if (mu < 0.5) {
        bp = 0.3, lo = p.lv[1], hi = p.lv[2];
    } else if (mu < 0.7) {
        bp = 0.5, lo = p.lv[2], hi = p.lv[3];
    } else {
        bp = 0.7, lo = p.lv[3], hi = p.lv[4];
    }
    const double t = __dmul_rn(5.0, __dsub_rn(mu, bp));
    alpha = __dadd_rn(lo, __dmul_rn(t, __dsub_rn(hi, lo)));
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

// ---------------------------------------------------------------- staging
// The CTA's cell neighbourhood in shared memory.  A CTA's 128 queries are
// consecutive in the block-major visiting order (query_key), so their cells
// form a compact patch; the patch widened by kStageMargin cells (the first
// block of a uniform k = 10 query is its 5 x 5 cells) is copied once —
// coordinates, ids and the local CSR offsets of every cell — and every row
// segment inside it is scanned from shared memory.  Segments outside it
// (wider blocks, rings) read global memory as before; which source a
// candidate comes from never changes the candidates or their order.
constexpr int kStageMargin = 2;
constexpr int kStagePts = 1536;   // 30 KB of {x, y, id}
constexpr int kStageCells = 1024; // local CSR entries (rows x (cols + 1))
constexpr int kStageRows = 64;

struct KnnStage {
    double2 xy[kStagePts];
    uint32_t id[kStagePts];
    uint32_t lcs[kStageCells];     // local offset of cell (r, c) of the patch, c in [C0, C1 + 1]
    uint32_t row_base[kStageRows + 1];
    uint32_t row_g[kStageRows];    // global CSR offset of the row segment's first point
    int r0, r1, c0, c1, on;
    int red[4][4];
};

// All threads of the CTA; valid: the thread holds a query at (row, col).
__device__ void stage_patch(const KnnArgs& a, KnnStage& st, bool valid, int row, int col) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int v[4] = {valid ? row : INT_MAX, valid ? -row : INT_MAX, valid ? col : INT_MAX,
                valid ? -col : INT_MAX};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] = min(v[i], __shfl_xor_sync(0xFFFFFFFFu, v[i], o));
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) st.red[warp][i] = v[i];
    __syncthreads();
    if (tid == 0) {
        int m[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
            for (int i = 0; i < 4; ++i) m[i] = min(m[i], st.red[w][i]);
        st.on = 0;
        if (m[0] != INT_MAX) {
            st.r0 = max(0, m[0] - kStageMargin), st.r1 = min(a.g.n_row - 1, -m[1] + kStageMargin);
            st.c0 = max(0, m[2] - kStageMargin), st.c1 = min(a.g.n_col - 1, -m[3] + kStageMargin);
            const int nr = st.r1 - st.r0 + 1, nc = st.c1 - st.c0 + 2;
            st.on = nr <= kStageRows && nr * nc <= kStageCells;
        }
    }
    __syncthreads();
    if (!st.on) return;
    const int nr = st.r1 - st.r0 + 1, nc = st.c1 - st.c0 + 2;  // nc: cells + 1 boundaries
    for (int i = tid; i < nr * nc; i += blockDim.x) {
        const int r = i / nc, c = i - r * nc;
        st.lcs[i] = __ldg(a.cell_start + static_cast<size_t>(st.r0 + r) * a.g.n_col + st.c0 + c);
    }
    __syncthreads();
    if (warp == 0) {  // row lengths -> exclusive prefix (rows <= 64: two warp passes)
        uint32_t carry = 0;
        for (int r0 = 0; r0 < nr; r0 += 32) {
            const int r = r0 + lane;
            const uint32_t len = r < nr ? st.lcs[r * nc + nc - 1] - st.lcs[r * nc] : 0u;
            uint32_t inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
                if (lane >= o) inc += t;
            }
            if (r < nr) {
                st.row_base[r] = carry + inc - len;
                st.row_g[r] = st.lcs[r * nc];
            }
            carry += __shfl_sync(0xFFFFFFFFu, inc, 31);
        }
        if (lane == 0) {
            st.row_base[nr] = carry;
            if (carry > static_cast<uint32_t>(kStagePts)) st.on = 0;
        }
    }
    __syncthreads();
    if (!st.on) return;
    for (int i = tid; i < nr * nc; i += blockDim.x) {  // global CSR -> local offsets
        const int r = i / nc;
        st.lcs[i] = st.row_base[r] + (st.lcs[i] - st.row_g[r]);
    }
    const uint32_t total = st.row_base[nr];
    for (uint32_t f = tid; f < total; f += blockDim.x) {
        int lo = 0, hi = nr - 1;  // the row holding local point f
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (st.row_base[mid] <= f) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t g = st.row_g[lo] + (f - st.row_base[lo]);
        st.xy[f] = __ldg(a.sorted_xy + g);
        st.id[f] = __ldg(a.sorted_ids + g);
    }
    __syncthreads();
}

// Points of row rr, cells [c0, c1] (clipped to the grid): contiguous in the
// cell-sorted arrays (row-major cells), so one cell_start round trip and one
// loop cover the whole segment.  Once the buffer is full the segment is
// trimmed to the cells whose padded rectangle can hold a point with
// d2 <= max(kth, snap_sq) — the per-cell lower bound of cell_lower_d2 solved
// for the column range, widened by a further safety margin (trimming only
// ever keeps more cells than the exact test, so results are unchanged).
// The next candidate's coordinates and id are loaded one iteration ahead.
template <class TopK>
__device__ __forceinline__ void scan_row(const KnnArgs& a, const KnnStage* st, TopK& t, double qx,
                                         double qy, double fx, double fy, double inv_w2, int rr,
                                         int c0, int c1, uint32_t& snap,
                                         unsigned long long& scanned) {
    const int n_col = a.g.n_col, n_row = a.g.n_row;
    if (t.full()) {
        const double inf = __longlong_as_double(0x7FF0000000000000ll);
        const double pad = 1.0e-7;
        const double thr = fmax(t.kth(), a.snap_sq);
        const double y0 = rr == 0 ? -inf : rr - pad, y1 = rr == n_row - 1 ? inf : rr + 1 + pad;
        const double dy = fmax(0.0, fmax(y0 - fy, fy - y1));
        // dx^2 budget in cell units; inv_w2 = 1 / (w2 (1 - 1e-9)) rounded up
        // by a further 1e-12, so room only ever errs high
        const double room = thr * inv_w2 - dy * dy;
        if (room < 0.0) return;  // the whole row is strictly worse
        // the reach in FP32 (MUFU sqrt), overestimated by 1e-5 relative +
        // 1e-4 cells: trimming keeps a superset of the exact test's cells
        const double h = static_cast<double>(sqrtf(__double2float_ru(room)) * 1.00001f + 1.0e-4f);
        // cell c is kept iff c - pad - fx <= h and fx - (c + 1 + pad) <= h;
        // the edge cells are unbounded outward (keep them on their open side)
        const double lo = floor(fx - h - pad - 1.0), hi = floor(fx + h + pad);
        int k0 = lo < c0 ? c0 : (lo > c1 ? c1 + 1 : static_cast<int>(lo));
        int k1 = hi > c1 ? c1 : (hi < c0 ? c0 - 1 : static_cast<int>(hi));
        if (c0 == 0 && k1 < 0) k1 = 0;
        if (c1 == n_col - 1 && k0 > n_col - 1) k0 = n_col - 1;
        c0 = k0, c1 = k1;
        if (c0 > c1) return;
    }
    if (st && rr >= st->r0 && rr <= st->r1 && c0 >= st->c0 && c1 <= st->c1) {
        const uint32_t* lcs = st->lcs + (rr - st->r0) * (st->c1 - st->c0 + 2) - st->c0;
        uint32_t s = lcs[c0];
        const uint32_t e = lcs[c1 + 1];
        scanned += e - s;
        for (; s < e; ++s) {
            const double2 cxy = st->xy[s];
            const uint32_t cid = st->id[s];
            const double cd = dsq_rn(qx, qy, cxy.x, cxy.y);
            if (cd <= a.snap_sq) snap = cid < snap ? cid : snap;
            if (t.admits(cd)) t.insert(cd, cid);
        }
        return;
    }
    const size_t base = static_cast<size_t>(rr) * static_cast<size_t>(n_col);
    uint32_t s = __ldg(a.cell_start + base + c0);
    const uint32_t e = __ldg(a.cell_start + base + c1 + 1);
    scanned += e - s;
    if (s >= e) return;
    double2 pxy = __ldg(a.sorted_xy + s);
    uint32_t pid = __ldg(a.sorted_ids + s);
    while (true) {
        const double2 cxy = pxy;
        const uint32_t cid = pid;
        const bool more = ++s < e;
        if (more) {
            pxy = __ldg(a.sorted_xy + s);
            pid = __ldg(a.sorted_ids + s);
        }
        const double cd = dsq_rn(qx, qy, cxy.x, cxy.y);
        if (cd <= a.snap_sq) snap = cid < snap ? cid : snap;
        if (t.admits(cd)) t.insert(cd, cid);
        if (!more) break;
    }
}

// One thread per query.
template <class TopK>
__global__ void __launch_bounds__(128) knn_grid_kernel(KnnArgs a) {
    __shared__ KnnStage stage;
    const size_t pos = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long scanned = 0, ref_scanned = 0;
    int col = 0, row = 0;
    if (pos < a.n) query_cell(a.qcell[pos], a.g.n_col, a.qkey_nbc, row, col);
    const KnnStage* stp = nullptr;
    if (a.stage) {
        stage_patch(a, stage, pos < a.n, row, col);
        if (stage.on) stp = &stage;
    }
    if (pos < a.n) {
        const uint32_t qi = a.perm[pos];
        const double qx = a.qx[qi], qy = a.qy[qi];
        const int n_col = a.g.n_col, n_row = a.g.n_row;

        // expansion level (knn.hpp:130-156)
        int level;
        if (a.m < static_cast<size_t>(a.k)) {
            level = imax(imax(col, n_col - 1 - col), imax(row, n_row - 1 - row));
        } else {
            // the smallest L0 whose clipped block holds >= k points: the
            // count is non-decreasing in L0 and reaches m >= k once the block
            // covers the grid, so a galloping search (L0 = 0, 1, 2, 4, ...)
            // then bisection finds exactly the reference's linear-scan L0 in
            // O(log L) block counts instead of O(L) (void queries of the
            // clustered stress case reach L ~ 100)
            const size_t kk = static_cast<size_t>(a.k);
            auto enough = [&](int L0) {
                return rect_count(a, imax(0, col - L0), imin(n_col - 1, col + L0),
                                  imax(0, row - L0), imin(n_row - 1, row + L0)) >= kk;
            };
            const int cover = imax(imax(col, n_col - 1 - col), imax(row, n_row - 1 - row));
            int lo = -1, hi = 0;  // invariant: !enough(lo) (lo = -1: vacuous), enough(hi)
            while (hi < cover && !enough(hi)) {
                lo = hi;
                hi = hi == 0 ? 1 : imin(2 * hi, cover);
            }
            while (hi - lo > 1) {
                const int mid = lo + (hi - lo) / 2;
                if (enough(mid)) hi = mid;
                else lo = mid;
            }
            level = hi + 1;
        }

        TopK t;
        t.init(a.k_eff, a.scratch_d + pos * a.k_eff, a.scratch_id + pos * a.k_eff);
        uint32_t snap = kNoId;
        // query in cell units, for the lower bounds
        const double fx = __ddiv_rn(__dsub_rn(qx, a.g.min_x), a.g.cell_width);
        const double fy = __ddiv_rn(__dsub_rn(qy, a.g.min_y), a.g.cell_width);
        const double w2 = __dmul_rn(a.g.cell_width, a.g.cell_width);
        const double inv_w2 = (1.0 / (w2 * (1.0 - 1.0e-9))) * (1.0 + 1.0e-12);
        // The reference scans the whole level block at once; scanning it row
        // by row outward from the query's row and trimming each row to the
        // cells that can still hold a point below the current k-th yields the
        // same k smallest (d2, idx) of the block, hence identical stop
        // decisions and results.
        {
            const int c0 = imax(0, col - level), c1 = imin(n_col - 1, col + level);
            for (int d = 0; d <= 2 * level; ++d) {
                const int rr = row + ((d & 1) ? -((d + 1) >> 1) : (d >> 1));
                if (rr < 0 || rr >= n_row) continue;
                scan_row(a, stp, t, qx, qy, fx, fy, inv_w2, rr, c0, c1, snap, scanned);
            }
        }
        // ring widening (knn.hpp:234-247, scan_ring :175-194)
        while (true) {
            const bool covers = col - level <= 0 && row - level <= 0 &&
                                col + level >= n_col - 1 && row + level >= n_row - 1;
            if (covers) break;
            const double reach = __dmul_rn(static_cast<double>(level), a.g.cell_width);
            const double bound = __dmul_rn(__dmul_rn(reach, reach), a.ring_margin);
            if (t.full() && t.kth() <= bound) break;
            ++level;
            const int r = level;
            const int c0 = imax(0, col - r), c1 = imin(n_col - 1, col + r);
            const int r0 = imax(0, row - r + 1), r1 = imin(n_row - 1, row + r - 1);
            // an empty ring (four O(1) block counts) or an empty side adds no
            // candidate: skipping it changes nothing but the cell lookups
            // (void queries of the stress case cross dozens of empty rings)
            if (a.rect_prefix &&
                rect_count(a, c0, c1, imax(0, row - r), imin(n_row - 1, row + r)) ==
                    rect_count(a, imax(0, col - r + 1), imin(n_col - 1, col + r - 1), r0, r1))
                continue;
            if (row - r >= 0) scan_row(a, stp, t, qx, qy, fx, fy, inv_w2, row - r, c0, c1, snap, scanned);
            if (row + r <= n_row - 1)
                scan_row(a, stp, t, qx, qy, fx, fy, inv_w2, row + r, c0, c1, snap, scanned);
            if (col - r >= 0 && (!a.rect_prefix || rect_count(a, col - r, col - r, r0, r1) > 0))
                for (int rr = r0; rr <= r1; ++rr)
                    scan_row(a, stp, t, qx, qy, fx, fy, inv_w2, rr, col - r, col - r, snap, scanned);
            if (col + r <= n_col - 1 && (!a.rect_prefix || rect_count(a, col + r, col + r, r0, r1) > 0))
                for (int rr = r0; rr <= r1; ++rr)
                    scan_row(a, stp, t, qx, qy, fx, fy, inv_w2, rr, col + r, col + r, snap, scanned);
        }
        if (a.ref_candidates) {  // what the reference scanned: the final-level block
            ref_scanned = rect_count(a, imax(0, col - level), imin(n_col - 1, col + level),
                                     imax(0, row - level), imin(n_row - 1, row + level));
        }
        finish_query(a, t, pos, qi, snap);
    }
    if (a.candidates) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            scanned += __shfl_xor_sync(0xFFFFFFFFu, scanned, o);
            ref_scanned += __shfl_xor_sync(0xFFFFFFFFu, ref_scanned, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (scanned) atomicAdd(a.candidates, scanned);
            if (a.ref_candidates && ref_scanned) atomicAdd(a.ref_candidates, ref_scanned);
        }
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

#define AIDW_KNN_CASE(KERNEL, K)                              \
    else if (a.k_eff <= K) {                                  \
        LAUNCH(KERNEL<RegTopK<K>>, blocks, 128, 0, s, a);     \
    }
#define AIDW_KNN_DISPATCH(KERNEL)                                   \
    do {                                                            \
        const unsigned blocks = ceil_div(a.n, 128);                 \
        if (a.k_eff <= 1) {                                         \
            LAUNCH(KERNEL<RegTopK<1>>, blocks, 128, 0, s, a);       \
        }                                                           \
        AIDW_KNN_CASE(KERNEL, 2) AIDW_KNN_CASE(KERNEL, 4)           \
        AIDW_KNN_CASE(KERNEL, 8) AIDW_KNN_CASE(KERNEL, 10)          \
        AIDW_KNN_CASE(KERNEL, 12) AIDW_KNN_CASE(KERNEL, 15)         \
        AIDW_KNN_CASE(KERNEL, 16)                                   \
        AIDW_KNN_CASE(KERNEL, 24) AIDW_KNN_CASE(KERNEL, 32)         \
        AIDW_KNN_CASE(KERNEL, 48) AIDW_KNN_CASE(KERNEL, 64)         \
        else {                                                      \
            LAUNCH(KERNEL<MemTopK>, blocks, 128, 0, s, a);          \
        }                                                           \
    } while (0)

}  // namespace

namespace {
// Summed-area table of the cell counts from the CSR prefix, stored column
// by column: PT[c][r] = points in rows < r, columns < c.  One CTA per column
// boundary c; its threads own contiguous row ranges (sum, block scan,
// rewrite): PT[c][r + 1] = PT[c][r] + (cell_start[r n_col + c] - cell_start[r n_col]).
constexpr int kPrefixThreads = 256;
__global__ void __launch_bounds__(kPrefixThreads) rect_prefix_kernel(
    const uint32_t* __restrict__ cell_start, int n_col, int n_row, uint32_t* __restrict__ PT) {
    __shared__ uint32_t warp_tot[kPrefixThreads / 32];
    const int c = blockIdx.x, t = threadIdx.x;
    const int per = (n_row + kPrefixThreads - 1) / kPrefixThreads;
    const int r0 = t * per, r1 = r0 + per < n_row ? r0 + per : n_row;
    auto row_count = [&](int r) {
        const size_t base = static_cast<size_t>(r) * static_cast<size_t>(n_col);
        return __ldg(cell_start + base + c) - __ldg(cell_start + base);
    };
    uint32_t sum = 0;
    for (int r = r0; r < r1; ++r) sum += row_count(r);
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if ((t & 31) >= o) inc += v;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = inc;
    __syncthreads();
    uint32_t before = inc - sum;
    for (int w = 0; w < (t >> 5); ++w) before += warp_tot[w];
    uint32_t* col = PT + static_cast<size_t>(c) * (static_cast<size_t>(n_row) + 1);
    if (t == 0) col[0] = 0;
    for (int r = r0; r < r1; ++r) {
        before += row_count(r);
        col[r + 1] = before;
    }
}
}  // namespace

void run_knn_grid(KnnArgs a, cudaStream_t s) {
    if (a.n == 0) return;
    static const int stage_env = [] {  // AIDW_K2_STAGE=0: no shared-memory staging (A/B)
        const char* v = std::getenv("AIDW_K2_STAGE");
        return v ? std::atoi(v) : 1;
    }();
    a.stage = a.stage && stage_env;
    DBuf<uint32_t> prefix;
    if (!a.rect_prefix && a.m >= static_cast<size_t>(a.k)) {
        prefix.alloc((static_cast<size_t>(a.g.n_row) + 1) * (static_cast<size_t>(a.g.n_col) + 1), s);
        LAUNCH(rect_prefix_kernel, static_cast<unsigned>(a.g.n_col) + 1, kPrefixThreads, 0, s,
               a.cell_start, a.g.n_col, a.g.n_row, prefix.get());
        a.rect_prefix = prefix.get();
    }
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
