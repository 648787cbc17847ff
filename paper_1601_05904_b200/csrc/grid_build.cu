// grid_build.cu — K1: even-grid construction on sm_100a.
//
// Replaces build_index (proj/include/aidw/grid.hpp:176-213): the reference
// runs a sequential counting sort (locate -> histogram -> prefix -> stable
// scatter).  Here the same CSR arrays come from
//   1. cell_ids_kernel  : FP64 locate_cell per point (exact reference
//                         rounding), key = row-major cell id, value = index,
//                         per-cell histogram with global atomics; two points
//                         per thread through double2 loads / uint2 stores;
//   2. exclusive_scan   : cell_start = exclusive prefix of the histogram
//                         (single pass, decoupled look-back);
//   3. counting sort    : scatter through per-cell atomic cursors, then each
//                         cell's ids sorted ascending (thread per point: rank in
//                         its cell of <= 16 points; warp rank placement up to 256, CTA bitonic up
//                         to 4096, stable compaction beyond) fused with the gather of the cell-sorted
//                         x / y.  (radix_sort_pairs — stable LSD, 8-bit digits,
//                         warp __match_any ranking — sorts the queries by cell.)
// All arrays are bit-identical to the reference's (tests/test_gpu_parity.py).
// Compiled with -fmad=false: every FP64 expression keeps the reference's
// two-rounding form.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace aidwb {

namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;  // per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys
constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;  // 2048 values

// Two points per thread: 16-byte (double2) coordinate loads and 8-byte
// (uint2) key / value stores when the arrays are aligned for them (device
// pointers handed in through aidw_run_pipeline_device may not be).
// key: the row-major cell id (nbc = 0; data points, histogrammed into
// counts) or the block-major query key (query_key)
__device__ __forceinline__ uint32_t cell_of(double x, double y, const GridGeom& g, size_t i,
                                            uint32_t* counts, long long* fail, int nbc) {
    int col, row;
    if (locate_cell_dev(x, y, g, col, row)) {
        const uint32_t cell = query_key(row, col, g.n_col, nbc);
        if (counts) atomicAdd(&counts[cell], 1u);
        return cell;
    }
    atomicMin(fail, static_cast<long long>(i));
    return 0;
}

template <bool VEC>
__global__ void cell_ids_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                size_t m, GridGeom g, uint32_t* __restrict__ keys,
                                uint32_t* __restrict__ vals, uint32_t* __restrict__ counts,
                                long long* __restrict__ fail, int nbc) {
    const size_t i = 2 * (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x);
    if (i >= m) return;
    if (VEC && i + 1 < m) {
        const double2 px = reinterpret_cast<const double2*>(x)[i / 2];
        const double2 py = reinterpret_cast<const double2*>(y)[i / 2];
        const uint32_t c0 = cell_of(px.x, py.x, g, i, counts, fail, nbc);
        const uint32_t c1 = cell_of(px.y, py.y, g, i + 1, counts, fail, nbc);
        reinterpret_cast<uint2*>(keys)[i / 2] = make_uint2(c0, c1);
        if (vals)
            reinterpret_cast<uint2*>(vals)[i / 2] =
                make_uint2(static_cast<uint32_t>(i), static_cast<uint32_t>(i + 1));
        return;
    }
    for (size_t j = i; j < i + 2 && j < m; ++j) {
        keys[j] = cell_of(x[j], y[j], g, j, counts, fail, nbc);
        if (vals) vals[j] = static_cast<uint32_t>(j);
    }
}

void launch_cell_ids(const double* x, const double* y, size_t m, const GridGeom& g,
                     uint32_t* keys, uint32_t* vals, uint32_t* counts, long long* fail,
                     cudaStream_t s, int nbc = 0) {
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(vals)) & 7) == 0;
    const size_t threads = ceil_div(m, static_cast<size_t>(2));
    if (vec)
        LAUNCH(cell_ids_kernel<true>, ceil_div(threads, kThreads), kThreads, 0, s, x, y, m, g,
               keys, vals, counts, fail, nbc);
    else
        LAUNCH(cell_ids_kernel<false>, ceil_div(threads, kThreads), kThreads, 0, s, x, y, m, g,
               keys, vals, counts, fail, nbc);
}

__global__ void interleave_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  size_t n, double2* __restrict__ xy) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) xy[i] = make_double2(x[i], y[i]);
}

// ---------------------------------------------------------------- scan
__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Single-pass exclusive scan (decoupled look-back): tiles of 2048 values are
// taken in ticket order; each warp scans 256 values (row-strided: element
// j * 32 + lane of its segment, so loads and stores are coalesced), the tile
// publishes its aggregate, then lane 0 of warp 0 walks back over the
// predecessors' (flag, value) words until an inclusive prefix is found.
// In place (in == out) is allowed: a tile reads all its values first.
constexpr unsigned long long kScanAggregate = 1ull << 32, kScanPrefix = 2ull << 32;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kThreads) scan_onepass_kernel(
    const uint32_t* in, uint32_t* out, size_t n, unsigned long long* __restrict__ status,
    unsigned* __restrict__ ticket, uint32_t* __restrict__ copy) {
    __shared__ unsigned s_tile;
    __shared__ uint32_t s_warp[kThreads / 32];
    __shared__ uint32_t s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = static_cast<size_t>(tile) * kScanTile + static_cast<size_t>(warp) * 32 * kScanItems;
    uint32_t v[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const size_t idx = base + static_cast<size_t>(j) * 32 + lane;
        v[j] = idx < n ? in[idx] : 0u;
    }
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const uint32_t inc = warp_inclusive_scan(v[j]);
        const uint32_t x = v[j];
        v[j] = run + inc - x;  // exclusive within the warp's segment
        run += __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
    if (lane == 0) s_warp[warp] = run;
    __syncthreads();
    if (warp == 0) {
        const uint32_t t = lane < kThreads / 32 ? s_warp[lane] : 0u;
        const uint32_t inc = warp_inclusive_scan(t);
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc, kThreads / 32 - 1);
        if (lane < kThreads / 32) s_warp[lane] = inc - t;
        // warp-wide look-back: lane l inspects tile (j - l) of a 32-tile
        // window; the window's aggregates are summed down to the nearest
        // inclusive prefix (tile -1 counts as an inclusive prefix of 0)
        if (lane == 0)
            st_release(&status[tile], (tile == 0 ? kScanPrefix : kScanAggregate) | total);
        uint32_t prefix = 0;
        for (long long jbase = static_cast<long long>(tile) - 1;;) {
            const long long jj = jbase - lane;
            const unsigned long long w = jj >= 0 ? ld_acquire(&status[jj]) : kScanPrefix;
            const unsigned pmask = __ballot_sync(0xFFFFFFFFu, (w & kScanPrefix) != 0);
            const int stop = pmask ? __ffs(pmask) - 1 : 31;
            // a tile up to the nearest prefix not published yet: look again
            if (__any_sync(0xFFFFFFFFu, lane <= stop && (w >> 32) == 0)) continue;
            uint32_t val = lane <= stop ? static_cast<uint32_t>(w) : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
            prefix += val;
            if (pmask) break;
            jbase -= 32;
        }
        if (lane == 0) {
            if (tile != 0) st_release(&status[tile], kScanPrefix | static_cast<uint32_t>(prefix + total));
            s_prefix = prefix;
        }
    }
    __syncthreads();
    const uint32_t add = s_prefix + s_warp[warp];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const size_t idx = base + static_cast<size_t>(j) * 32 + lane;
        if (idx < n) {
            out[idx] = v[j] + add;
            if (copy) copy[idx] = v[j] + add;
        }
    }
}

// ---------------------------------------------------------------- radix sort
// Per tile: histogram of the digit -> hist[digit * tiles + tile].
__global__ void radix_upsweep_kernel(const uint32_t* __restrict__ keys, size_t n, int shift,
                                     uint32_t* __restrict__ hist, unsigned tiles) {
    __shared__ uint32_t h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(blockIdx.x) * kSortTile;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const size_t idx = base + static_cast<size_t>(j) * kSortThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & (kRadix - 1)], 1u);
    }
    __syncthreads();
    hist[static_cast<size_t>(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: warp w owns keys [tile + w*256, +256), taken 32 at a time
// in index order; a key's rank = (same digit in earlier warps) + (same digit
// in earlier rounds of this warp) + (same digit in lower lanes this round).
__global__ void radix_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                     const uint32_t* __restrict__ vals_in,
                                     uint32_t* __restrict__ keys_out,
                                     uint32_t* __restrict__ vals_out, size_t n, int shift,
                                     const uint32_t* __restrict__ offsets, unsigned tiles) {
    __shared__ uint32_t cnt[kSortWarps][kRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) cnt[w][threadIdx.x] = 0;
    __syncthreads();

    const size_t base = static_cast<size_t>(blockIdx.x) * kSortTile +
                        static_cast<size_t>(warp) * (32 * kSortItems);
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const size_t idx = base + static_cast<size_t>(r) * 32 + lane;
        const bool valid = idx < n;
        k[r] = valid ? keys_in[idx] : 0u;
        v[r] = valid ? vals_in[idx] : 0u;
        const uint32_t d = valid ? ((k[r] >> shift) & (kRadix - 1)) : kRadix;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        const uint32_t before = valid ? cnt[warp][d] : 0u;
        rank[r] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (valid && (__ffs(peers) - 1) == lane) cnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = cnt[w][threadIdx.x];
            cnt[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const size_t idx = base + static_cast<size_t>(r) * 32 + lane;
        if (idx < n) {
            const uint32_t d = (k[r] >> shift) & (kRadix - 1);
            const size_t pos = static_cast<size_t>(offsets[static_cast<size_t>(d) * tiles + blockIdx.x]) +
                               cnt[warp][d] + rank[r];
            keys_out[pos] = k[r];
            vals_out[pos] = v[r];
        }
    }
}

// ---------------------------------------------------------------- min / max
__device__ __forceinline__ unsigned long long order_key(double d) {
    const unsigned long long u = as_u64(d);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

// keys[0..2] = min x, y, z ; keys[3..5] = max x, y, z (order-preserving u64
// encoding; NaNs are skipped like std::min/max in compute_bbox).
__global__ void minmax_kernel(const double* __restrict__ ax, const double* __restrict__ ay,
                              size_t na, const double* __restrict__ bx,
                              const double* __restrict__ by, size_t nb,
                              const double* __restrict__ z, size_t nz,
                              unsigned long long* __restrict__ keys) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t start = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t total = na + nb;
    for (size_t i = start; i < total; i += stride) {
        const double x = i < na ? ax[i] : bx[i - na];
        const double y = i < na ? ay[i] : by[i - na];
        if (x == x) {
            const unsigned long long kx = order_key(x);
            lo[0] = kx < lo[0] ? kx : lo[0];
            hi[0] = kx > hi[0] ? kx : hi[0];
        }
        if (y == y) {
            const unsigned long long ky = order_key(y);
            lo[1] = ky < lo[1] ? ky : lo[1];
            hi[1] = ky > hi[1] ? ky : hi[1];
        }
    }
    for (size_t i = start; i < nz; i += stride) {
        const double v = z[i];
        if (v == v) {
            const unsigned long long kz = order_key(v);
            lo[2] = kz < lo[2] ? kz : lo[2];
            hi[2] = kz > hi[2] ? kz : hi[2];
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        lo[q] = warp_min_u64(lo[q]);
        hi[q] = warp_max_u64(hi[q]);
    }
    // CTA reduction first: one atomic per key per CTA (per-warp atomics on
    // the same six words serialise in L2)
    __shared__ unsigned long long s_k[6][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) s_k[q][warp] = lo[q], s_k[3 + q][warp] = hi[q];
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = static_cast<int>(blockDim.x >> 5);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            lo[q] = warp_min_u64(lane < nw ? s_k[q][lane] : ~0ull);
            hi[q] = warp_max_u64(lane < nw ? s_k[3 + q][lane] : 0ull);
        }
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            atomicMin(&keys[q], lo[q]);
            atomicMax(&keys[3 + q], hi[q]);
        }
    }
}

__global__ void decode_minmax_kernel(const unsigned long long* __restrict__ keys,
                                     double* __restrict__ out6) {
    // out6 = {min_x, min_y, max_x, max_y, min_z, max_z}
    const int map[6] = {0, 1, 3, 4, 2, 5};
    const int t = threadIdx.x;
    if (t < 6) {
        const unsigned long long k = keys[map[t]];
        const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
        out6[t] = __longlong_as_double(static_cast<long long>(u));
    }
}

// ---------------------------------------------------------------- counting sort
// The CSR arrays of build_index as a counting sort (grid.hpp:176-213 is one
// too): histogram (cell_ids_kernel) -> exclusive scan (cell_start) ->
// scatter through per-cell atomic cursors (order within a cell arbitrary) ->
// each cell's ids sorted ascending, which is exactly the reference's stable
// order, fused with the coordinate gather.  Points of cells of <= kSmallCell
// points are placed by one thread each (rank among the cell's ids), cells up
// to kMidCell by a warp, larger ones by a CTA (cell_sort_big_kernel).
constexpr int kSmallCell = 16;
constexpr int kMidCell = 256;
constexpr int kBigCell = 4096;

__global__ void cell_scatter_kernel(const uint32_t* __restrict__ keys, size_t m,
                                    uint32_t* __restrict__ cursor, uint32_t* __restrict__ ids) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) ids[atomicAdd(&cursor[keys[i]], 1u)] = static_cast<uint32_t>(i);
}

__device__ __forceinline__ void emit_point(size_t s, uint32_t id, const double* __restrict__ x,
                                           const double* __restrict__ y, uint32_t* __restrict__ ids,
                                           double2* __restrict__ sxy, double* __restrict__ sx,
                                           double* __restrict__ sy) {
    const double px = x[id], py = y[id];
    ids[s] = id;
    sxy[s] = make_double2(px, py);
    if (sx) {
        sx[s] = px;
        sy[s] = py;
    }
}

// One thread per scattered position: a point of a cell of <= kSmallCell
// points is placed by its rank among the cell's ids (ids are distinct, so the
// ascending order is the reference's stable order), fused with the gather.
// The first position of a larger cell queues it for the warp / CTA kernels.
__global__ void cell_rank_small_kernel(const uint32_t* __restrict__ cell_start,
                                       const uint32_t* __restrict__ keys, size_t m,
                                       const uint32_t* __restrict__ scattered,
                                       const double* __restrict__ x, const double* __restrict__ y,
                                       uint32_t* __restrict__ ids, double2* __restrict__ sxy,
                                       double* __restrict__ sx, double* __restrict__ sy,
                                       uint32_t* __restrict__ mid, uint32_t* __restrict__ big,
                                       uint32_t* __restrict__ nbig) {
    const size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const uint32_t id = scattered[p];
    const uint32_t c = keys[id];
    const uint32_t b = cell_start[c], e = cell_start[c + 1];
    const uint32_t n = e - b;
    if (n > kSmallCell) {  // nbig[0]: warp-sized cells, nbig[1]: CTA-sized
        if (p == b) {
            if (n <= kMidCell) mid[atomicAdd(&nbig[0], 1u)] = c;
            else big[atomicAdd(&nbig[1], 1u)] = c;
        }
        return;
    }
    uint32_t rank = 0;
    for (uint32_t q = b; q < e; ++q) rank += scattered[q] < id ? 1u : 0u;
    emit_point(b + rank, id, x, y, ids, sxy, sx, sy);
}

// One warp per queued cell of kSmallCell < n <= kMidCell points: the ids go
// to a per-warp shared buffer and each lane places its ids by rank (the
// number of smaller ids in the cell; ids are distinct), then the gather.
__device__ __forceinline__ void sort_mid_cells(
    unsigned block, unsigned nblocks, uint32_t (*buf)[kMidCell],
    const uint32_t* __restrict__ cell_start, const uint32_t* __restrict__ mid,
    const uint32_t* __restrict__ nmid, const uint32_t* __restrict__ scattered,
    const double* __restrict__ x, const double* __restrict__ y, uint32_t* __restrict__ ids,
    double2* __restrict__ sxy, double* __restrict__ sx, double* __restrict__ sy) {
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const uint32_t warps = nblocks * (blockDim.x >> 5);
    for (uint32_t w = block * (blockDim.x >> 5) + wp; w < *nmid; w += warps) {
        const uint32_t c = mid[w];
        const uint32_t b = cell_start[c], n = cell_start[c + 1] - b;
        for (uint32_t j = lane; j < n; j += 32) buf[wp][j] = scattered[b + j];
        __syncwarp();
        for (uint32_t j = lane; j < n; j += 32) {
            const uint32_t mine = buf[wp][j];
            uint32_t rank = 0;
            for (uint32_t k = 0; k < n; ++k) rank += buf[wp][k] < mine ? 1u : 0u;
            emit_point(b + rank, mine, x, y, ids, sxy, sx, sy);
        }
        __syncwarp();
    }
}

// One CTA per queued cell (n > kMidCell): a bitonic sort of the ids in
// shared memory (padded with 0xFFFFFFFF) when n <= kBigCell, then the
// gather.  A cell above kBigCell (degenerate, heavily duplicated data) is
// instead rebuilt by a stable compaction of the key array in index order —
// O(m) for that cell, correct for any size, no host round trip.
__device__ __forceinline__ void sort_big_cells(
    unsigned block, unsigned nblocks, uint32_t* v, uint32_t* wsum,
    const uint32_t* __restrict__ cell_start, const uint32_t* __restrict__ big,
    const uint32_t* __restrict__ nbig, const uint32_t* __restrict__ scattered,
    const uint32_t* __restrict__ keys, size_t m, const double* __restrict__ x,
    const double* __restrict__ y, uint32_t* __restrict__ ids, double2* __restrict__ sxy,
    double* __restrict__ sx, double* __restrict__ sy) {
    for (uint32_t w = block; w < *nbig; w += nblocks) {
        const uint32_t c = big[w];
        const uint32_t b = cell_start[c], n = cell_start[c + 1] - b;
        __syncthreads();
        if (n > static_cast<uint32_t>(kBigCell)) {
            uint32_t run = 0;  // points of cell c before this chunk (all threads)
            for (size_t base = 0; base < m; base += blockDim.x) {
                const size_t i = base + threadIdx.x;
                const bool hit = i < m && keys[i] == c;
                const unsigned ball = __ballot_sync(0xFFFFFFFFu, hit);
                const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
                if (lane == 0) wsum[wp] = __popc(ball);
                __syncthreads();
                uint32_t before = run, total = run;
                for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) {
                    if (k < wp) before += wsum[k];
                    total += wsum[k];
                }
                if (hit) {
                    const uint32_t s = b + before + __popc(ball & ((1u << lane) - 1u));
                    emit_point(s, static_cast<uint32_t>(i), x, y, ids, sxy, sx, sy);
                }
                run = total;
                __syncthreads();
            }
            continue;
        }
        uint32_t len = 1;
        while (len < n) len <<= 1;
        for (uint32_t j = threadIdx.x; j < len; j += blockDim.x)
            v[j] = j < n ? scattered[b + j] : 0xFFFFFFFFu;
        __syncthreads();
        for (uint32_t size = 2; size <= len; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) {
                    const uint32_t partner = j ^ stride;
                    if (partner > j) {
                        const bool up = (j & size) == 0;
                        const uint32_t a = v[j], o = v[partner];
                        if ((a > o) == up) {
                            v[j] = o;
                            v[partner] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x)
            emit_point(b + j, v[j], x, y, ids, sxy, sx, sy);
    }
}

// One launch for both crowded-cell queues: CTAs [0, kMidCtas) take the
// warp-sized cells, the rest the CTA-sized ones (role uniform per CTA).
constexpr unsigned kMidCtas = 148u * 4u, kBigCtas = 148u * 2u;
__global__ void __launch_bounds__(256) cell_sort_crowded_kernel(
    const uint32_t* __restrict__ cell_start, const uint32_t* __restrict__ mid,
    const uint32_t* __restrict__ big, const uint32_t* __restrict__ nbig,
    const uint32_t* __restrict__ scattered, const uint32_t* __restrict__ keys, size_t m,
    const double* __restrict__ x, const double* __restrict__ y, uint32_t* __restrict__ ids,
    double2* __restrict__ sxy, double* __restrict__ sx, double* __restrict__ sy) {
    __shared__ uint32_t buf[8][kMidCell];
    __shared__ uint32_t v[kBigCell];
    __shared__ uint32_t wsum[8];
    if (blockIdx.x < kMidCtas)
        sort_mid_cells(blockIdx.x, kMidCtas, buf, cell_start, mid, nbig, scattered, x, y, ids,
                       sxy, sx, sy);
    else
        sort_big_cells(blockIdx.x - kMidCtas, gridDim.x - kMidCtas, v, wsum, cell_start, big,
                       nbig + 1, scattered, keys, m, x, y, ids, sxy, sx, sy);
}

// Blocked cell order (K4 data tiles): cells visited in 8 x 8-cell blocks,
// blocks row-major, cells row-major inside a block.  On a factor-4 grid a
// block holds ~256 points (16 r_exp^2 m / A = 4 points per cell), so a
// 256-record K4 tile is a compact square instead of a 64-cell strip.
constexpr int kOrderBlock = 8;

__device__ __forceinline__ bool block_slot_cell(size_t j, int n_col, int n_row, unsigned nbc,
                                                size_t& cell) {
    const size_t b = j / (kOrderBlock * kOrderBlock);
    const int w = static_cast<int>(j % (kOrderBlock * kOrderBlock));
    const size_t row = (b / nbc) * kOrderBlock + w / kOrderBlock;
    const size_t col = (b % nbc) * kOrderBlock + w % kOrderBlock;
    if (row >= static_cast<size_t>(n_row) || col >= static_cast<size_t>(n_col)) return false;
    cell = row * static_cast<size_t>(n_col) + col;
    return true;
}

__global__ void block_counts_kernel(const uint32_t* __restrict__ cell_start, int n_col, int n_row,
                                    unsigned nbc, size_t slots, uint32_t* __restrict__ cnt) {
    const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= slots) return;
    size_t c;
    cnt[j] = block_slot_cell(j, n_col, n_row, nbc, c) ? cell_start[c + 1] - cell_start[c] : 0u;
}

__global__ void block_scatter_kernel(const uint32_t* __restrict__ cell_start,
                                     const uint32_t* __restrict__ sorted_ids, int n_col, int n_row,
                                     unsigned nbc, size_t slots, const uint32_t* __restrict__ start,
                                     uint32_t* __restrict__ order) {
    const size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= slots) return;
    size_t c;
    if (!block_slot_cell(j, n_col, n_row, nbc, c)) return;
    const uint32_t b = cell_start[c], e = cell_start[c + 1], o = start[j];
    for (uint32_t t = b; t < e; ++t) order[o + (t - b)] = sorted_ids[t];
}

int bits_for(uint64_t max_key) {
    int b = 0;
    while (b < 32 && (max_key >> b) != 0) ++b;
    return b;
}

}  // namespace

void exclusive_scan_u32(const uint32_t* d_in, uint32_t* d_out, size_t n, cudaStream_t s,
                        uint32_t* d_copy) {
    if (n == 0) return;
    const unsigned tiles = ceil_div(n, kScanTile);
    // status words (one per tile) + the tile ticket, zeroed together
    DBuf<unsigned long long> status(static_cast<size_t>(tiles) + 1, s);
    CK(cudaMemsetAsync(status.get(), 0, (static_cast<size_t>(tiles) + 1) * sizeof(unsigned long long), s));
    LAUNCH(scan_onepass_kernel, tiles, kThreads, 0, s, d_in, d_out, n, status.get(),
           reinterpret_cast<unsigned*>(status.get() + tiles), d_copy);
}

void radix_sort_pairs(uint32_t* keys, uint32_t* vals, size_t n, int bits, cudaStream_t s) {
    if (n <= 1 || bits <= 0) return;
    const int passes = (bits + kRadixBits - 1) / kRadixBits;
    const unsigned tiles = ceil_div(n, kSortTile);
    DBuf<uint32_t> k2(n, s), v2(n, s), hist(static_cast<size_t>(kRadix) * tiles, s);
    uint32_t *ki = keys, *vi = vals, *ko = k2.get(), *vo = v2.get();
    for (int p = 0; p < passes; ++p) {
        const int shift = p * kRadixBits;
        LAUNCH(radix_upsweep_kernel, tiles, kSortThreads, 0, s, ki, n, shift, hist.get(), tiles);
        exclusive_scan_u32(hist.get(), hist.get(), static_cast<size_t>(kRadix) * tiles, s);
        LAUNCH(radix_scatter_kernel, tiles, kSortThreads, 0, s, ki, vi, ko, vo, n, shift,
               hist.get(), tiles);
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    if (ki != keys) {
        CK(cudaMemcpyAsync(keys, ki, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(vals, vi, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    }
}

void blocked_cell_order(const uint32_t* d_cell_start, const uint32_t* d_sorted_ids, int n_col,
                        int n_row, size_t m, uint32_t* d_order, cudaStream_t s) {
    if (m == 0) return;
    const unsigned nbc = static_cast<unsigned>((n_col + kOrderBlock - 1) / kOrderBlock);
    const size_t nbr = static_cast<size_t>((n_row + kOrderBlock - 1) / kOrderBlock);
    const size_t slots = nbr * nbc * kOrderBlock * kOrderBlock;
    DBuf<uint32_t> cnt(slots, s);
    LAUNCH(block_counts_kernel, ceil_div(slots, kThreads), kThreads, 0, s, d_cell_start, n_col,
           n_row, nbc, slots, cnt.get());
    exclusive_scan_u32(cnt.get(), cnt.get(), slots, s);
    LAUNCH(block_scatter_kernel, ceil_div(slots, kThreads), kThreads, 0, s, d_cell_start,
           d_sorted_ids, n_col, n_row, nbc, slots, cnt.get(), d_order);
}

void interleave_xy(const double* d_x, const double* d_y, size_t n, double2* d_xy,
                   cudaStream_t s) {
    if (n) LAUNCH(interleave_kernel, ceil_div(n, kThreads), kThreads, 0, s, d_x, d_y, n, d_xy);
}

void build_grid_device(const double* d_x, const double* d_y, size_t m,
                       const aidw_grid_config& cfg, DeviceGrid& out, long long* d_fail,
                       cudaStream_t s, bool split_coords) {
    const GridGeom g = make_geom(cfg);
    const size_t cells = static_cast<size_t>(cfg.n_col) * static_cast<size_t>(cfg.n_row);
    out.cfg = cfg;
    out.m = m;
    out.cells = cells;
    out.cell_start.alloc(cells + 1, s);
    out.sorted_ids.alloc(m, s);
    out.sorted_xy.alloc(m, s);
    if (split_coords) {
        out.sorted_x.alloc(m, s);
        out.sorted_y.alloc(m, s);
    }
    DBuf<uint32_t> keys(m, s), vals(m, s), cursor(cells + 1, s), mid(cells, s), big(cells, s),
        nbig(2, s);
    CK(cudaMemsetAsync(out.cell_start.get(), 0, (cells + 1) * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(nbig.get(), 0, 2 * sizeof(uint32_t), s));
    launch_cell_ids(d_x, d_y, m, g, keys.get(), nullptr, out.cell_start.get(), d_fail, s);
    // counting sort: cursors start at cell_start (written by the same scan,
    // cells + 1 entries); vals receives the scatter
    exclusive_scan_u32(out.cell_start.get(), out.cell_start.get(), cells + 1, s, cursor.get());
    LAUNCH(cell_scatter_kernel, ceil_div(m, kThreads), kThreads, 0, s, keys.get(), m,
           cursor.get(), vals.get());
    LAUNCH(cell_rank_small_kernel, ceil_div(m, kThreads), kThreads, 0, s,
           out.cell_start.get(), keys.get(), m, vals.get(), d_x, d_y, out.sorted_ids.get(),
           out.sorted_xy.get(), out.sorted_x.get(), out.sorted_y.get(), mid.get(), big.get(),
           nbig.get());
    LAUNCH(cell_sort_crowded_kernel, kMidCtas + kBigCtas, 256, 0, s, out.cell_start.get(),
           mid.get(), big.get(), nbig.get(), vals.get(), keys.get(), m, d_x, d_y,
           out.sorted_ids.get(), out.sorted_xy.get(), out.sorted_x.get(), out.sorted_y.get());
}

int sort_queries_by_cell(const double* d_qx, const double* d_qy, size_t n, const GridGeom& g,
                         DBuf<uint32_t>& perm, DBuf<uint32_t>& cells, long long* d_fail,
                         cudaStream_t s) {
    perm.alloc(n, s);
    cells.alloc(n, s);
    const int nbc = query_block_cols(g.n_col, g.n_row);
    if (n == 0) return nbc;
    launch_cell_ids(d_qx, d_qy, n, g, cells.get(), perm.get(), nullptr, d_fail, s, nbc);
    const size_t total = nbc ? static_cast<size_t>(nbc) * ((static_cast<size_t>(g.n_row) + 7) >> kQBlockBits) * 64
                             : static_cast<size_t>(g.n_col) * static_cast<size_t>(g.n_row);
    // the cell order only buys locality (every query's result is independent
    // of the visiting order): few queries are bucketed by their key's top bits
    // in one launch instead of the six of the two radix passes
    if (n <= small_sort_n()) bucket_by_key_small(cells.get(), perm.get(), n, bits_for(total - 1), s);
    else radix_sort_pairs(cells.get(), perm.get(), n, bits_for(total - 1), s);
    return nbc;
}

// One CTA groups up to kSmallSortMax (key, value) pairs by the top B <= 12
// bits of their `bits`-bit keys (counting sort through 2^B shared counters;
// the order inside a bucket is unspecified — callers use it for locality
// only).  Loads are issued kUnroll at a time: a lone CTA is latency-bound.
constexpr int kBucketMaxBits = 12;
constexpr int kBucketThreads = 1024;
constexpr int kUnroll = 8;
constexpr size_t kSmallSortMax = 65536;
constexpr size_t kBucketSmemMax = 200 * 1024;  // counters + copies in shared memory up to this
// SMEM: the (key, value) copies stay in shared memory after the counters
// (n small enough), else in the global scratch tk / tv.
template <bool SMEM>
__global__ void __launch_bounds__(kBucketThreads) bucket_small_kernel(uint32_t* __restrict__ keys,
                                                                      uint32_t* __restrict__ vals,
                                                                      size_t n, int shift, int nb,
                                                                      uint32_t* __restrict__ tk,
                                                                      uint32_t* __restrict__ tv) {
    extern __shared__ uint32_t cnt[];  // nb = 2^B counters (then 2n copies if SMEM)
    __shared__ uint32_t wsum[kBucketThreads / 32];
    if (SMEM) {
        tk = cnt + nb;
        tv = tk + n;
    }
    const int t = threadIdx.x;
    for (int b = t; b < nb; b += kBucketThreads) cnt[b] = 0u;
    __syncthreads();
    for (size_t i0 = 0; i0 < n; i0 += static_cast<size_t>(kUnroll) * kBucketThreads) {
        uint32_t k[kUnroll], v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t i = i0 + static_cast<size_t>(u) * kBucketThreads + t;
            k[u] = i < n ? keys[i] : 0u;
            v[u] = i < n ? vals[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t i = i0 + static_cast<size_t>(u) * kBucketThreads + t;
            if (i < n) {
                tk[i] = k[u], tv[i] = v[u];
                atomicAdd(&cnt[k[u] >> shift], 1u);
            }
        }
    }
    __syncthreads();
    // exclusive scan of the counters: a contiguous run per thread, warp
    // shuffles, then the warp totals
    const int per = nb / kBucketThreads > 0 ? nb / kBucketThreads : 1;
    const int b0 = t * per;
    uint32_t run = 0;
    for (int j = 0; j < per; ++j) run += b0 + j < nb ? cnt[b0 + j] : 0u;
    uint32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if ((t & 31) >= o) inc += x;
    }
    if ((t & 31) == 31) wsum[t >> 5] = inc;
    __syncthreads();
    if (t < 32) {
        const uint32_t w = wsum[t];
        uint32_t winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, winc, o);
            if (t >= o) winc += x;
        }
        wsum[t] = winc - w;
    }
    __syncthreads();
    uint32_t base = wsum[t >> 5] + inc - run;
    for (int j = 0; j < per; ++j)
        if (b0 + j < nb) {
            const uint32_t c = cnt[b0 + j];
            cnt[b0 + j] = base;
            base += c;
        }
    __syncthreads();
    for (size_t i0 = 0; i0 < n; i0 += static_cast<size_t>(kUnroll) * kBucketThreads) {
        uint32_t k[kUnroll], v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t i = i0 + static_cast<size_t>(u) * kBucketThreads + t;
            k[u] = i < n ? tk[i] : 0u;
            v[u] = i < n ? tv[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const size_t i = i0 + static_cast<size_t>(u) * kBucketThreads + t;
            if (i < n) {
                const uint32_t pos = atomicAdd(&cnt[k[u] >> shift], 1u);
                keys[pos] = k[u], vals[pos] = v[u];
            }
        }
    }
}

void bucket_by_key_small(uint32_t* keys, uint32_t* vals, size_t n, int bits, cudaStream_t s) {
    if (n == 0) return;
    if (n > kSmallSortMax) {
        radix_sort_pairs(keys, vals, n, bits, s);
        return;
    }
    const int b = bits < kBucketMaxBits ? (bits > 1 ? bits : 1) : kBucketMaxBits;
    const int shift = bits - b;
    const int nb = 1 << b;
    const size_t smem = static_cast<size_t>(nb) * sizeof(uint32_t);
    const size_t smem_all = smem + 2 * n * sizeof(uint32_t);
    if (smem_all <= kBucketSmemMax) {  // the copies in shared memory: no global round trip
        CK(cudaFuncSetAttribute(bucket_small_kernel<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_all)));
        LAUNCH(bucket_small_kernel<true>, 1, kBucketThreads, smem_all, s, keys, vals, n, shift, nb,
               static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr));
        return;
    }
    CK(cudaFuncSetAttribute(bucket_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    DBuf<uint32_t> tk(n, s), tv(n, s);
    LAUNCH(bucket_small_kernel<false>, 1, kBucketThreads, smem, s, keys, vals, n, shift, nb,
           tk.get(), tv.get());
}

size_t small_sort_n() {
    static const size_t v = [] {  // AIDW_SMALL_SORT_N: tuning / A-B
        const char* e = std::getenv("AIDW_SMALL_SORT_N");
        return e ? static_cast<size_t>(std::atoll(e)) : static_cast<size_t>(65536);
    }();
    return v;
}

void bbox_reduce_device(const double* d_ax, const double* d_ay, size_t na, const double* d_bx,
                        const double* d_by, size_t nb, const double* d_z, size_t nz,
                        double* d_out6, cudaStream_t s) {
    DBuf<unsigned long long> keys(6, s);
    CK(cudaMemsetAsync(keys.get(), 0xFF, 3 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(keys.get() + 3, 0, 3 * sizeof(unsigned long long), s));
    const size_t total = na + nb > nz ? na + nb : nz;
    // one value per thread while that fits 148 x 8 CTAs (a small reduction is
    // load-latency-bound: no thread should wait on a chain of loads)
    unsigned blocks = ceil_div(total ? total : 1, kThreads);
    if (blocks > 148u * 8u) blocks = 148u * 8u;
    LAUNCH(minmax_kernel, blocks, kThreads, 0, s, d_ax, d_ay, na, d_bx, d_by, nb, d_z, nz,
           keys.get());
    LAUNCH(decode_minmax_kernel, 1, 32, 0, s, keys.get(), d_out6);
}

}  // namespace aidwb
