// common.cuh — shared device helpers, launch accounting and the workspace
// allocator of the B200 AIDW library.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "aidw_capi.h"

namespace aidwb {

// ------------------------------------------------------------------ errors
struct Failure : std::exception {
    int code;
    long long index;
    std::string msg;
    Failure(int c, std::string m, long long i = -1) : code(c), index(i), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw Failure(AIDW_ERR_CUDA, std::string("CUDA error in ") + what + " (" + file + ":" +
                                         std::to_string(line) + "): " + cudaGetErrorString(e));
    }
}
#define CK(x) ::aidwb::cuda_check((x), #x, __FILE__, __LINE__)

// Every kernel launch of the library goes through LAUNCH so the launch
// counter (aidw_kernel_launch_count, bench.py's gpu_launches) is exact.
extern std::atomic<long long> g_launches;
// While a pass is being captured into a CUDA graph its launches are counted
// here (they run when the graph is launched, and are counted then).
extern thread_local long long* t_launch_sink;
#define LAUNCH(kernel, grid, block, smem, stream, ...)                                   \
    do {                                                                                 \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                      \
        if (::aidwb::t_launch_sink) ++*::aidwb::t_launch_sink;                            \
        else ::aidwb::g_launches.fetch_add(1, std::memory_order_relaxed);                \
        CK(cudaGetLastError());                                                          \
    } while (0)

// Timing event on a stream.  During CUDA-graph capture it becomes an
// external event-record node (so graph replays still time); the external
// flag is rejected outside capture, so it is used only then.
inline void record_event(cudaEvent_t e, cudaStream_t s) {
    if (!e) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &st));
    if (st == cudaStreamCaptureStatusActive)
        CK(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else
        CK(cudaEventRecord(e, s));
}

// ------------------------------------------------------------------ workspace
// Stream-ordered device buffers.  Inside a pipeline call (ArenaScope in
// capi.cu) they are bump-allocated from one cached per-call workspace on the
// call's stream — no allocator API call per buffer, no reuse within the call
// (so no aliasing); the workspace is recycled only after the call's stream
// has synchronised.  Elsewhere, or when the workspace is full, they come
// from the default memory pool (kept warm by a release threshold set once per
// device, see capi.cu).
struct Arena {
    char* base = nullptr;
    size_t cap = 0, used = 0, overflow = 0;
    unsigned small = 0;  // consecutive calls that used < 1/8 of a large workspace
    cudaStream_t stream = nullptr;
};
extern thread_local Arena* t_arena;

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    bool pooled = true;  // false: carved from the call's arena
    DBuf() = default;
    DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    void alloc(size_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (!count) return;
        const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        Arena* a = t_arena;
        if (a && a->stream == stream) {
            if (a->used + bytes <= a->cap) {
                p = reinterpret_cast<T*>(a->base + a->used);
                a->used += bytes;
                pooled = false;
                return;
            }
            a->overflow += bytes;  // grow the workspace for the next call
        }
        CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
    }
    void release() {
        if (p && pooled) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
        pooled = true;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    T* get() const { return p; }
    operator T*() const { return p; }
};

// ------------------------------------------------------------------ geometry
// Grid geometry with the host-precomputed locate_cell bounds
// (grid.hpp:93-106: fx in [-slack, n + slack], slack = 1e-9 * (n + 1)).
struct GridGeom {
    double cell_width;
    int n_col, n_row;
    double min_x, min_y;
    double lo_x, hi_x, lo_y, hi_y;
};

// Query visiting order of K2: cells in 8 x 8-cell blocks, blocks row-major,
// cells row-major inside a block, so 128 consecutive queries cover a compact
// square of cells (row-major cell ids give a one-row strip).  nbc = blocks
// per grid row; 0 = plain row-major ids (key range would not fit 32 bits).
constexpr int kQBlockBits = 3;
inline int query_block_cols(int n_col, int n_row) {
    const uint64_t nbc = (static_cast<uint64_t>(n_col) + 7) >> kQBlockBits;
    const uint64_t nbr = (static_cast<uint64_t>(n_row) + 7) >> kQBlockBits;
    return nbc * nbr * 64 <= 0xFFFFFFFFull ? static_cast<int>(nbc) : 0;
}
__host__ __device__ __forceinline__ uint32_t query_key(int row, int col, int n_col, int nbc) {
    if (nbc == 0) return static_cast<uint32_t>(row) * static_cast<uint32_t>(n_col) + static_cast<uint32_t>(col);
    const uint32_t b = static_cast<uint32_t>(row >> kQBlockBits) * static_cast<uint32_t>(nbc) +
                       static_cast<uint32_t>(col >> kQBlockBits);
    return (b << (2 * kQBlockBits)) | (static_cast<uint32_t>(row & 7) << kQBlockBits) |
           static_cast<uint32_t>(col & 7);
}
__host__ __device__ __forceinline__ void query_cell(uint32_t key, int n_col, int nbc, int& row,
                                                    int& col) {
    if (nbc == 0) {
        col = static_cast<int>(key % static_cast<uint32_t>(n_col));
        row = static_cast<int>(key / static_cast<uint32_t>(n_col));
        return;
    }
    const uint32_t b = key >> (2 * kQBlockBits);
    row = static_cast<int>((b / static_cast<uint32_t>(nbc)) << kQBlockBits) + static_cast<int>((key >> kQBlockBits) & 7);
    col = static_cast<int>((b % static_cast<uint32_t>(nbc)) << kQBlockBits) + static_cast<int>(key & 7);
}

inline GridGeom make_geom(const aidw_grid_config& c) {
    GridGeom g;
    g.cell_width = c.cell_width;
    g.n_col = c.n_col;
    g.n_row = c.n_row;
    g.min_x = c.min_x;
    g.min_y = c.min_y;
    const double sx = 1.0e-9 * (static_cast<double>(c.n_col) + 1.0);
    const double sy = 1.0e-9 * (static_cast<double>(c.n_row) + 1.0);
    g.lo_x = -sx;
    g.hi_x = static_cast<double>(c.n_col) + sx;
    g.lo_y = -sy;
    g.hi_y = static_cast<double>(c.n_row) + sy;
    return g;
}

// Squared distance with the reference's exact rounding sequence
// (knn.hpp:23-27 under -ffp-contract=off): two products, then one add.
__device__ __forceinline__ double dsq_rn(double qx, double qy, double px, double py) {
    const double dx = __dsub_rn(px, qx);
    const double dy = __dsub_rn(py, qy);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// locate_cell (grid.hpp:93-106): FP64 divide, slack test, floor, clamp.
// Returns false when the point lies outside the covered region (or is NaN).
__device__ __forceinline__ bool locate_cell_dev(double x, double y, const GridGeom& g, int& col,
                                                int& row) {
    const double fx = __ddiv_rn(__dsub_rn(x, g.min_x), g.cell_width);
    const double fy = __ddiv_rn(__dsub_rn(y, g.min_y), g.cell_width);
    if (!(fx >= g.lo_x && fx <= g.hi_x) || !(fy >= g.lo_y && fy <= g.hi_y)) return false;
    int c = static_cast<int>(floor(fx));
    int r = static_cast<int>(floor(fy));
    c = c < 0 ? 0 : (c > g.n_col - 1 ? g.n_col - 1 : c);
    r = r < 0 ? 0 : (r > g.n_row - 1 ? g.n_row - 1 : r);
    col = c;
    row = r;
    return true;
}

__device__ __forceinline__ unsigned long long as_u64(double d) {
    return static_cast<unsigned long long>(__double_as_longlong(d));
}

constexpr uint32_t kNoId = 0xFFFFFFFFu;
constexpr int kThreads = 256;

inline unsigned ceil_div(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// ------------------------------------------------------------------ host decls
// grid_build.cu
struct DeviceGrid {
    aidw_grid_config cfg;
    size_t m = 0, cells = 0;
    DBuf<uint32_t> cell_start;  // cells + 1
    DBuf<uint32_t> sorted_ids;  // m
    DBuf<double> sorted_x, sorted_y;  // API outputs (only when requested)
    DBuf<double2> sorted_xy;          // interleaved copy the kNN kernel reads
};

// order[0..m) = the grid's point ids with cells visited in 8 x 8-cell blocks
// (blocks row-major, cells row-major inside): compact K4 data tiles.
void blocked_cell_order(const uint32_t* d_cell_start, const uint32_t* d_sorted_ids, int n_col,
                        int n_row, size_t m, uint32_t* d_order, cudaStream_t s);

// Builds the CSR grid from device x/y (m points).  Out-of-region points
// set *d_fail (atomicMin of the point index); the caller checks it.
void build_grid_device(const double* d_x, const double* d_y, size_t m,
                       const aidw_grid_config& cfg, DeviceGrid& out, long long* d_fail,
                       cudaStream_t s, bool split_coords = false);

// xy[i] = {x[i], y[i]}
void interleave_xy(const double* d_x, const double* d_y, size_t n, double2* d_xy, cudaStream_t s);

// Sort n query points by cell: returns the permutation (sorted position ->
// query index) and the sorted query keys (query_key, block-major cells);
// the result is the keys' nbc (blocks per grid row); failures -> *d_fail.
int sort_queries_by_cell(const double* d_qx, const double* d_qy, size_t n, const GridGeom& g,
                          DBuf<uint32_t>& perm, DBuf<uint32_t>& cells, long long* d_fail,
                          cudaStream_t s);

// Generic exclusive scan of n uint32 values (in place allowed).
void exclusive_scan_u32(const uint32_t* d_in, uint32_t* d_out, size_t n, cudaStream_t s,
                        uint32_t* d_copy = nullptr);

// Stable LSD radix sort of (key, value) u32 pairs on the low `bits` bits.
void radix_sort_pairs(uint32_t* keys, uint32_t* vals, size_t n, int bits, cudaStream_t s);
// Queries up to this count take a one-launch bucketing (top 12 key bits) for
// the locality orders (cell order for K2, Morton order for K4) instead of
// the radix sort: visiting order never changes a result (AIDW_SMALL_SORT_N).
size_t small_sort_n();
void bucket_by_key_small(uint32_t* keys, uint32_t* vals, size_t n, int bits, cudaStream_t s);

// min/max reductions: out[0..3] = bbox(a ∪ b) (x,y), optional z hull out[4..5]
void bbox_reduce_device(const double* d_ax, const double* d_ay, size_t na, const double* d_bx,
                        const double* d_by, size_t nb, const double* d_z, size_t nz,
                        double* d_out6, cudaStream_t s);

}  // namespace aidwb
