// capi.cu — the extern "C" entry points (include/aidw_capi.h) and the fused,
// device-resident run_pipeline.
//
// Host code here only validates, computes the reference's scalar set-up
// (cell width, grid geometry, r_exp, snap tolerance — with the reference's
// own expressions, compiled with -ffp-contract=off) and orchestrates the
// sm_100a kernels of grid_build.cu (K1), knn.cu (K2 + K3) and weight.cu /
// weight64.cu (K4).  No per-query arithmetic of the hot path runs on the
// host; without a CUDA device every entry point fails with AIDW_ERR_CUDA.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <new>
#include <numbers>
#include <string>
#include <vector>

#include "aidw_capi.h"
#include "common.cuh"
#include "knn.cuh"
#include "replicate.cuh"
#include "weight.cuh"

namespace aidwb {

std::atomic<long long> g_launches{0};
thread_local long long* t_launch_sink = nullptr;
thread_local Arena* t_arena = nullptr;

namespace {

std::atomic<int> g_precision{[] {
    const char* e = std::getenv("AIDW_WEIGHT_FP64");
    return (e && e[0] == '1') ? AIDW_PRECISION_FP64 : AIDW_PRECISION_FP32;
}()};

// ------------------------------------------------------------ host set-up
// The reference's scalar expressions (types.hpp, grid.hpp, adaptive.hpp,
// interpolate.hpp), evaluated on the host exactly as written there.
struct Box {
    double min_x, min_y, max_x, max_y;
    double width() const { return max_x - min_x; }
    double height() const { return max_y - min_y; }
    double area() const { return width() * height(); }
    bool valid() const { return min_x <= max_x && min_y <= max_y; }
    bool degenerate() const { return !(area() > 0.0); }
};

double choose_cell_width_h(size_t m, const Box& b, double factor) {  // grid.hpp:50-64
    if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "choose_cell_width: data set is empty");
    if (!b.valid() || b.degenerate())
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "choose_cell_width: bbox must have positive area");
    if (!(factor > 0.0) || !std::isfinite(factor))
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "choose_cell_width: factor must be positive finite");
    const double density = static_cast<double>(m) / b.area();
    return factor * (1.0 / (2.0 * std::sqrt(density)));
}

aidw_grid_config make_grid_config_h(const Box& b, double w) {  // grid.hpp:67-88
    if (!b.valid() || b.degenerate())
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "make_grid_config: bbox must have positive area");
    if (!(w > 0.0) || !std::isfinite(w))
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "make_grid_config: cellWidth must be positive finite");
    const double cols = std::floor((b.max_x - b.min_x + w) / w);
    const double rows = std::floor((b.max_y - b.min_y + w) / w);
    if (cols * rows > 1.0e9)
        throw Failure(AIDW_ERR_INVALID_ARGUMENT,
                      "make_grid_config: cellWidth " + std::to_string(w) + " yields more than 1e9 cells");
    aidw_grid_config c;
    c.cell_width = w;
    c.n_col = std::max(1, static_cast<int>(cols));
    c.n_row = std::max(1, static_cast<int>(rows));
    c.min_x = b.min_x;
    c.min_y = b.min_y;
    return c;
}

void validate_params(const aidw_params& p) {  // types.hpp:102-114
    if (p.k < 1)
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "AidwParams: k must be >= 1, got " + std::to_string(p.k));
    if (!(p.r_min < p.r_max)) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "AidwParams: rMin must be < rMax");
    for (double a : p.alpha_levels)
        if (!(a > 0.0) || !std::isfinite(a))
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "AidwParams: alpha levels must be positive finite");
}

AlphaParams alpha_params_h(const aidw_params& p, double r_exp) {
    AlphaParams a;
    a.r_exp = r_exp;
    a.pi_over_rmax = std::numbers::pi / p.r_max;  // adaptive.hpp:59
    a.r_min = p.r_min;
    a.r_max = p.r_max;
    for (int i = 0; i < 5; ++i) a.lv[i] = p.alpha_levels[i];
    return a;
}

double snap_sq_h(const Box& b) {  // interpolate.hpp:86-89
    const double eps = 1.0e-12 * std::hypot(b.width(), b.height());
    return eps * eps;
}

// d_zhull: the device value hull {zlo, zhi} (the kernels derive zshift).
WeightFrame make_frame(const Box& b, const double* d_zhull) {
    WeightFrame f;
    f.ox = b.min_x;
    f.oy = b.min_y;
    const double span = std::max(b.width(), b.height());
    f.inv_scale = (span > 0.0 && std::isfinite(span)) ? 1.0 / span : 1.0;
    f.zhull = d_zhull;
    f.snap_sq = snap_sq_h(b);
    return f;
}

std::string locate_msg(double x, double y) {  // grid.hpp:100-101
    return "locate_cell: point (" + std::to_string(x) + ", " + std::to_string(y) +
           ") lies outside the covered region";
}

// AIDW_HOST_TRACE=1: host-side phase times of each fused pass on stderr.
bool host_trace() {
    static const bool on = [] {
        const char* v = std::getenv("AIDW_HOST_TRACE");
        return v && *v == '1';
    }();
    return on;
}

// ------------------------------------------------------------ device context
std::once_flag g_pool_once[64];
size_t g_pool_keep[64];  // the pool's release threshold per device
std::once_flag g_pinned_once;
void* pinned_alloc(size_t bytes);
void pinned_free(void* p);

int current_device() {
    static std::atomic<int> known{0};  // the device count, asked until a device is found
    if (known.load(std::memory_order_relaxed) == 0) {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            throw Failure(AIDW_ERR_CUDA, std::string("no CUDA device available: ") +
                                              (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
        known.store(count, std::memory_order_relaxed);
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::call_once(g_pool_once[dev & 63], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            // Reserve a working set once (up to 8 GiB of freed memory stays
            // in the pool), so later calls never pay pool growth inside a
            // timed stage; memory freed beyond it goes back at sync points.
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
                const size_t want = std::min<size_t>(free_b / 8, size_t(8) << 30);
                uint64_t thr = want;
                g_pool_keep[dev & 63] = want;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                void* p = nullptr;
                if (want && cudaMallocAsync(&p, want, 0) == cudaSuccess) {
                    cudaFreeAsync(p, 0);
                    cudaStreamSynchronize(0);
                }
            }
        }
    });
    // one 64 MiB page-locked staging block for the drop-in's result copies,
    // pinned once per process at first device use
    std::call_once(g_pinned_once, [] { pinned_free(pinned_alloc(1)); });
    return dev;
}

// The stream of a call: the caller's, or (stream == NULL) the library's own
// non-blocking stream for this host thread and device — created once and
// kept (creating and destroying one per call cost ~50 us, an eighth of a
// 10K x 10K pass); a call on it is synchronous (the stream is drained
// before the call returns) and starts after the work already queued on the
// legacy default stream (e.g. the caller's cudaMemcpyAsync(..., 0) of a
// device input): one event recorded there, waited on by the library's stream.
struct ManagedStreams {
    cudaStream_t s[64] = {};
    cudaEvent_t legacy[64] = {};
    ~ManagedStreams() {  // thread exit: no stream outlives its thread
        for (int i = 0; i < 64; ++i) {
            if (s[i]) cudaStreamDestroy(s[i]);
            if (legacy[i]) cudaEventDestroy(legacy[i]);
        }
    }
};
cudaStream_t managed_stream(int dev) {
    thread_local ManagedStreams streams;
    cudaStream_t& s = streams.s[dev & 63];
    cudaEvent_t& e = streams.legacy[dev & 63];
    if (!s) {
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(e, cudaStreamLegacy));
    CK(cudaStreamWaitEvent(s, e, 0));
    return s;
}

// A pair of timing events for this host thread and the current device
// (the uploads of aidw_run_pipeline), created once.
struct ThreadEvents {
    cudaEvent_t b[64] = {}, e[64] = {};
    ~ThreadEvents() {
        for (int i = 0; i < 64; ++i) {
            if (b[i]) cudaEventDestroy(b[i]);
            if (e[i]) cudaEventDestroy(e[i]);
        }
    }
};
void h2d_events(cudaEvent_t& b, cudaEvent_t& e) {
    thread_local ThreadEvents ev;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!ev.b[dev & 63]) CK(cudaEventCreate(&ev.b[dev & 63]));
    if (!ev.e[dev & 63]) CK(cudaEventCreate(&ev.e[dev & 63]));
    b = ev.b[dev & 63];
    e = ev.e[dev & 63];
}

struct StreamScope {
    cudaStream_t s = nullptr;
    bool own = false;
    explicit StreamScope(void* external = nullptr) {
        const int dev = current_device();
        if (external) {
            s = static_cast<cudaStream_t>(external);
        } else {
            s = managed_stream(dev);
            own = true;
        }
    }
    void sync() { CK(cudaStreamSynchronize(s)); }
    ~StreamScope() {
        if (own) cudaStreamSynchronize(s);
    }
};

struct Events {
    std::vector<cudaEvent_t> ev;
    cudaEvent_t make() {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ev.push_back(e);
        return e;
    }
    static double ms(cudaEvent_t a, cudaEvent_t b) {
        float t = 0.f;
        if (a && b) {
            if (cudaEventElapsedTime(&t, a, b) == cudaSuccess) return t;
            cudaGetLastError();  // stage never ran (e.g. n == 0): clear, do not leak
        }
        return 0.0;
    }
    ~Events() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

template <typename T>
void h2d(DBuf<T>& dst, const T* src, size_t n, cudaStream_t s) {
    dst.alloc(n, s);
    if (n) CK(cudaMemcpyAsync(dst.get(), src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <typename T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n && dst) CK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

// bbox of (a ∪ b) plus the z hull, device reduce -> host.
// d_out6 = {min_x, min_y, max_x, max_y, zlo, zhi} of (a ∪ b) and z.
struct Extents {
    Box box;
    const double* d_hull = nullptr;  // device, 6 doubles; zhull = d_hull + 4
};
// Device reduce into d_out6, then (one host round trip) the box.
Extents extents(double* d_out6, const double* ax, const double* ay, size_t na, const double* bx,
                const double* by, size_t nb, const double* z, size_t nz, cudaStream_t s) {
    bbox_reduce_device(ax, ay, na, bx, by, nb, z, nz, d_out6, s);
    double h[6];
    d2h(h, d_out6, 6, s);
    CK(cudaStreamSynchronize(s));
    return Extents{Box{h[0], h[1], h[2], h[3]}, d_out6};
}
// Host box only (the device result is dropped with the call).
Box extents_box(const double* ax, const double* ay, size_t na, const double* bx,
                const double* by, size_t nb, cudaStream_t s) {
    DBuf<double> out(6, s);
    return extents(out.get(), ax, ay, na, bx, by, nb, nullptr, 0, s).box;
}

// Slots 0-2: failure indices (LLONG_MAX = none); 3-5: counters (0).
__global__ void fail_init_kernel(long long* __restrict__ d) {
    if (threadIdx.x < 8) d[threadIdx.x] = threadIdx.x < 3 ? LLONG_MAX : 0;
}

// Failure indices written by kernels (atomicMin), resolved after sync, and
// the pass's device counters (recipe queries, kNN candidates) in the same
// 64-byte block, so one copy returns everything.  Initialised on the stream
// by a one-warp kernel (no host round trip).
struct FailFlags {
    DBuf<long long> d;
    long long h[8];
    explicit FailFlags(cudaStream_t s, bool defer_init = false) : d(8, s) {
        for (int i = 0; i < 8; ++i) h[i] = i < 3 ? LLONG_MAX : 0;
        if (!defer_init) init(s);
    }
    void init(cudaStream_t s) { LAUNCH(fail_init_kernel, 1, 32, 0, s, d.get()); }
    long long* slot(int i) { return d.get() + i; }
    unsigned long long* counter(int i) { return reinterpret_cast<unsigned long long*>(d.get() + i); }
    void fetch(cudaStream_t s) {
        d2h(h, d.get(), 8, s);
        CK(cudaStreamSynchronize(s));
    }
};
enum { kFailData = 0, kFailQuery = 1, kFailAlpha = 2, kCountAlpha4 = 3, kCountCand = 4,
       kCountRefCand = 5 };

void record(cudaEvent_t e, cudaStream_t s) { record_event(e, s); }

// Device-side nearest / snap search for the weighting stage when no kNN
// stage ran (idw mode and the aidw_predict_all drop-in).  Uses a k = 1 grid
// search (K1 + K2), or the brute kernel for tiny / degenerate sets.
struct NearestInfo {
    DeviceGrid grid;      // factor-4 grid (kept alive: its cell order feeds K4)
    DBuf<uint32_t> perm;  // visiting order
    DBuf<double> d2min;
    DBuf<uint32_t> nn, snap;
};

void nearest_search(const double* d_dx, const double* d_dy, size_t m, const double* d_qx,
                    const double* d_qy, size_t n, const Box& box, double snap_sq,
                    NearestInfo& out, FailFlags& fails, cudaStream_t s) {
    out.d2min.alloc(n, s);
    out.nn.alloc(n, s);
    out.snap.alloc(n, s);
    KnnArgs a;
    a.qx = d_qx;
    a.qy = d_qy;
    a.n = n;
    a.m = m;
    a.k = 1;
    a.k_eff = 1;
    a.snap_sq = snap_sq;
    a.d2min_s = out.d2min.get();
    a.nn_s = out.nn.get();
    a.snap_s = out.snap.get();
    bool use_grid = m > 4096 && box.valid() && !box.degenerate() && std::isfinite(box.area());
    aidw_grid_config cfg{};
    if (use_grid) {
        try {
            cfg = make_grid_config_h(box, choose_cell_width_h(m, box, 4.0));
        } catch (const Failure&) {
            use_grid = false;
        }
    }
    if (!use_grid) {
        out.perm.alloc(0, s);
        a.dx = d_dx;
        a.dy = d_dy;
        run_knn_brute(a, s);
        return;
    }
    DeviceGrid& g = out.grid;
    build_grid_device(d_dx, d_dy, m, cfg, g, fails.slot(kFailData), s);
    DBuf<uint32_t> qcell;
    const GridGeom geom = make_geom(cfg);
    const int nbc = sort_queries_by_cell(d_qx, d_qy, n, geom, out.perm, qcell, fails.slot(kFailQuery), s);
    a.g = geom;
    a.cell_start = g.cell_start.get();
    a.sorted_ids = g.sorted_ids.get();
    a.sorted_xy = g.sorted_xy.get();
    a.perm = out.perm.get();
    a.qcell = qcell.get();
    a.qkey_nbc = nbc;
    run_knn_grid(a, s);
}

// Device "alpha by visiting position" = gather of alpha-by-query.
__global__ void gather_f64_kernel(const double* __restrict__ src, const uint32_t* __restrict__ perm,
                                  size_t n, double* __restrict__ dst) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm ? perm[i] : i];
}
__global__ void fill_f64_kernel(double* __restrict__ dst, size_t n, double v) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = v;
}

// Which weighting kernel a (variant, pinned_order) call runs.
enum class WeightMode { fp32, fp64_blocked, fp64_naive };
WeightMode weight_mode(int32_t variant, int32_t pinned) {
    if (variant == AIDW_VARIANT_NAIVE || pinned != 0) return WeightMode::fp64_naive;
    return g_precision.load(std::memory_order_relaxed) == AIDW_PRECISION_FP64
               ? WeightMode::fp64_blocked
               : WeightMode::fp32;
}

// Weighting stage over device-resident inputs given alpha by query index.
void set_order(WeightData& wd, const DeviceGrid& g) {
    wd.order = g.sorted_ids.get();
    wd.cell_start = g.cell_start.get();
    wd.n_col = g.cfg.n_col;
    wd.n_row = g.cfg.n_row;
}

// d_alpha_q: alpha per query (input order).
void weighting_stage(const double* d_dx, const double* d_dy, const double* d_dz, size_t m,
                     const double* d_qx, const double* d_qy, size_t n, const double* d_alpha_q,
                     const Extents& ext, WeightMode mode, double* d_pred, double* d_alpha_out,
                     FailFlags& fails, WeightTimes* wt, cudaStream_t s) {
    const WeightFrame frame = make_frame(ext.box, ext.d_hull + 4);
    WeightData wd{d_dx, d_dy, d_dz, m};
    // snap index, nearest index and d2_min per query (k = 1 grid search,
    // FP64): the weighting kernels' snap rule and non-finite fallback
    NearestInfo nb;
    nearest_search(d_dx, d_dy, m, d_qx, d_qy, n, ext.box, frame.snap_sq, nb, fails, s);
    const uint32_t* perm = nb.perm.n ? nb.perm.get() : nullptr;
    if (nb.grid.sorted_ids.n) set_order(wd, nb.grid);
    DBuf<double> alpha_s(n, s);
    LAUNCH(gather_f64_kernel, ceil_div(n, kThreads), kThreads, 0, s, d_alpha_q, perm, n,
           alpha_s.get());
    WeightQueries q;
    q.qx = d_qx;
    q.qy = d_qy;
    q.n = n;
    q.perm = perm;
    q.alpha_s = alpha_s.get();
    q.d2min_s = nb.d2min.get();
    q.nn_s = nb.nn.get();
    q.snap_s = nb.snap.get();
    if (mode != WeightMode::fp32)
        weighting_fp64(q, wd, frame, mode == WeightMode::fp64_blocked, d_pred, d_alpha_out, wt, s);
    else
        weighting_fp32(q, wd, frame, d_pred, d_alpha_out, wt, s);
}

void fill_error(aidw_error* err, int code, const std::string& msg, long long index) {
    if (!err) return;
    err->code = code;
    err->index = index;
    std::strncpy(err->message, msg.c_str(), sizeof(err->message) - 1);
    err->message[sizeof(err->message) - 1] = '\0';
}

template <class F>
int guarded(aidw_error* err, F&& body) {
    if (err) fill_error(err, AIDW_OK, "", -1);
    cudaGetLastError();  // our static runtime: drop any stale error from an earlier call
    try {
        body();
        return AIDW_OK;
    } catch (const Failure& f) {
        fill_error(err, f.code, f.msg, f.index);
        return f.code;
    } catch (const std::bad_alloc&) {
        fill_error(err, AIDW_ERR_RUNTIME, "host allocation failed", -1);
        return AIDW_ERR_RUNTIME;
    } catch (const std::exception& e) {
        fill_error(err, AIDW_ERR_RUNTIME, e.what(), -1);
        return AIDW_ERR_RUNTIME;
    }
}

// ------------------------------------------------------------ pipeline core
struct PipelineIO {
    const double *dx, *dy, *dz, *qx, *qy;  // device
    size_t m, n;
    double *pred, *alpha;                  // device
};

// Timing events of one fused pass (stage marks, kNN kernel, K4 launches).
struct PassEvents {
    cudaEvent_t build0 = nullptr, build1 = nullptr, knn1 = nullptr, interp1 = nullptr;
    cudaEvent_t knnb = nullptr, knne = nullptr, k4b = nullptr, k4e = nullptr;
    void create() {
        for (cudaEvent_t* e : {&build0, &build1, &knn1, &interp1, &knnb, &knne, &k4b, &k4e})
            CK(cudaEventCreate(e));
    }
    void destroy() {
        for (cudaEvent_t* e : {&build0, &build1, &knn1, &interp1, &knnb, &knne, &k4b, &k4e}) {
            if (*e) cudaEventDestroy(*e);
            *e = nullptr;
        }
    }
};

// Every host-side scalar of a fused pass (the reference's set-up
// expressions), computed before any device work is enqueued: the kernels
// receive only these, so a pass with the same plan and buffers is the same
// sequence of launches (what the CUDA-graph cache relies on).
struct PassPlan {
    bool idw = false;
    Extents ext{};
    aidw_params params{};  // k clamped to m
    WeightMode wmode = WeightMode::fp32;
    aidw_grid_config gc{};  // the kNN grid (grid engine)
    double r_exp = 0.0;
    WeightFrame frame{};
    bool own_g4 = false;  // K4 record order from a separate factor-4 grid
    aidw_grid_config g4c{};
    double* d_hull = nullptr;   // device {bbox, zlo, zhi}
    bool hull_in_pass = false;  // reduce the value hull as the pass's first step
};

// Validation + extents (the one host round trip before the pass) + set-up
// (cli.hpp:217-268, with the reference's exception order).
PassPlan plan_pass(const PipelineIO& io, const aidw_run_config& cfg, aidw_run_stats* st,
                   double* d_hull, cudaStream_t s) {
    if (cfg.workers < 0)
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "resolve_workers: worker count must be >= 0");
    const size_t m = io.m, n = io.n;
    if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set is empty");
    if (!io.dz) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set carries no values");
    PassPlan pl;
    pl.wmode = weight_mode(cfg.variant, 0);
    // bbox(data ∪ queries) and the value hull.  A given bbox needs no host
    // round trip: the value hull is reduced inside the pass (device only).
    if (cfg.use_bbox) {
        pl.ext = Extents{Box{cfg.bbox[0], cfg.bbox[1], cfg.bbox[2], cfg.bbox[3]}, d_hull};
        pl.hull_in_pass = true;
    } else {
        pl.ext = extents(d_hull, io.dx, io.dy, m, io.qx, io.qy, n, io.dz, m, s);
    }
    pl.d_hull = d_hull;
    pl.frame = make_frame(pl.ext.box, d_hull + 4);
    if (cfg.mode == AIDW_MODE_IDW) {
        if (!(cfg.alpha > 0.0) || !std::isfinite(cfg.alpha))
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "idw_predict_all: alpha must be positive finite");
        pl.idw = true;
        if (st) st->k_effective = 0;
        return pl;
    }
    // k clamp (cli.hpp:237-238): the reference converts k to size_t first,
    // so a negative k clamps to m as well.
    pl.params = cfg.params;
    pl.params.k = static_cast<int32_t>(
        std::min<size_t>(static_cast<size_t>(static_cast<int64_t>(cfg.params.k)), m));
    if (st) st->k_effective = pl.params.k;
    const double area = pl.params.area > 0.0 ? pl.params.area : pl.ext.box.area();
    // the reference's order (cli.hpp:240-259): the grid engine's cell width
    // rejects a zero-area bbox (invalid_argument) before any query runs; the
    // per-query area failure of aidw_predict_all needs a query to fail on
    if (cfg.engine == AIDW_ENGINE_GRID)
        pl.gc = make_grid_config_h(pl.ext.box, choose_cell_width_h(m, pl.ext.box, cfg.cell_factor));
    validate_params(pl.params);  // aidw_predict_all's params.validate() (interpolate.hpp:457)
    if (n > 0 && (!(area > 0.0) || !std::isfinite(area)))
        throw Failure(AIDW_ERR_RUNTIME,
                      "aidw_predict_all: query 0: expected_nn_distance: area must be positive finite", 0);
    pl.r_exp = 1.0 / (2.0 * std::sqrt(static_cast<double>(m) / area));  // adaptive.hpp:27
    // K4 record order: cell order of the factor-4 grid over the bbox — the
    // kNN grid when it is one, else built for K4 — so the FP32 sums depend on
    // the inputs only, never on the kNN engine or cell factor
    if (pl.wmode == WeightMode::fp32 && m > 4096 &&  // same rule as nearest_search
        !(cfg.engine == AIDW_ENGINE_GRID && cfg.cell_factor == 4.0)) {
        try {
            pl.g4c = make_grid_config_h(pl.ext.box, choose_cell_width_h(m, pl.ext.box, 4.0));
            pl.own_g4 = true;
        } catch (const Failure&) {
            pl.own_g4 = false;
        }
    }
    return pl;
}

// The device work of one fused pass (cli.hpp:217-268): no host round trip,
// no allocation outside the call's workspace (when it fits).
void enqueue_pass(const PassPlan& pl, const PipelineIO& io, const aidw_run_config& cfg,
                  const PassEvents& pe, FailFlags& fails, cudaStream_t s) {
    const size_t m = io.m, n = io.n;
    if (pl.hull_in_pass)
        bbox_reduce_device(nullptr, nullptr, 0, nullptr, nullptr, 0, io.dz, m, pl.d_hull, s);
    WeightTimes wt;
    wt.k4_begin = pe.k4b;
    wt.k4_end = pe.k4e;
    wt.d_alpha4 = fails.counter(kCountAlpha4);
    if (pl.idw) {
        record(pe.build0, s);
        record(pe.build1, s);
        record(pe.knn1, s);
        DBuf<double> alpha_q(n, s);
        if (n) LAUNCH(fill_f64_kernel, ceil_div(n, kThreads), kThreads, 0, s, alpha_q.get(), n, cfg.alpha);
        weighting_stage(io.dx, io.dy, io.dz, m, io.qx, io.qy, n, alpha_q.get(), pl.ext, pl.wmode,
                        io.pred, io.alpha, fails, &wt, s);
        record(pe.interp1, s);
        return;
    }
    const int k = pl.params.k;
    KnnArgs a;
    a.qx = io.qx;
    a.qy = io.qy;
    a.n = n;
    a.m = m;
    a.k = k;
    a.k_eff = k;
    a.candidates = fails.counter(kCountCand);
    a.ref_candidates = fails.counter(kCountRefCand);
    a.snap_sq = pl.frame.snap_sq;
    a.compute_alpha = 1;
    a.ap = alpha_params_h(pl.params, pl.r_exp);
    a.fail_alpha = fails.slot(kFailAlpha);
    DBuf<double> alpha_s(n, s), d2min_s(n, s);
    DBuf<uint32_t> nn_s(n, s), snap_s(n, s), perm, qcell;
    a.alpha_s = alpha_s.get();
    a.d2min_s = d2min_s.get();
    a.nn_s = nn_s.get();
    a.snap_s = snap_s.get();
    DeviceGrid g;  // lives until the weighting stage has read its cell order
    if (cfg.engine == AIDW_ENGINE_GRID) {
        record(pe.build0, s);
        build_grid_device(io.dx, io.dy, m, pl.gc, g, fails.slot(kFailData), s);
        record(pe.build1, s);
        const GridGeom geom = make_geom(pl.gc);
        a.qkey_nbc = sort_queries_by_cell(io.qx, io.qy, n, geom, perm, qcell, fails.slot(kFailQuery), s);
        a.g = geom;
        a.cell_start = g.cell_start.get();
        a.sorted_ids = g.sorted_ids.get();
        a.sorted_xy = g.sorted_xy.get();
        a.perm = perm.get();
        a.qcell = qcell.get();
        record(pe.knnb, s);
        run_knn_grid(a, s);
        record(pe.knne, s);
        record(pe.knn1, s);
    } else {
        record(pe.build0, s);
        record(pe.build1, s);
        a.dx = io.dx;
        a.dy = io.dy;
        record(pe.knnb, s);
        run_knn_brute(a, s);
        record(pe.knne, s);
        record(pe.knn1, s);
    }
    WeightData wd{io.dx, io.dy, io.dz, m};
    DeviceGrid g4;
    if (pl.wmode == WeightMode::fp32 && m > 4096) {
        if (pl.own_g4) {
            build_grid_device(io.dx, io.dy, m, pl.g4c, g4, fails.slot(kFailData), s);
            set_order(wd, g4);
        } else if (cfg.engine == AIDW_ENGINE_GRID && cfg.cell_factor == 4.0) {
            set_order(wd, g);
        }
    }
    WeightQueries q;
    q.qx = io.qx;
    q.qy = io.qy;
    q.n = n;
    q.perm = perm.n ? perm.get() : nullptr;
    q.alpha_s = alpha_s.get();
    q.d2min_s = d2min_s.get();
    q.nn_s = nn_s.get();
    q.snap_s = snap_s.get();
    if (pl.wmode != WeightMode::fp32)
        weighting_fp64(q, wd, pl.frame, pl.wmode == WeightMode::fp64_blocked, io.pred, io.alpha, &wt, s);
    else
        weighting_fp32(q, wd, pl.frame, io.pred, io.alpha, &wt, s);
    record(pe.interp1, s);
}

// The reference's exceptions for the failures the pass recorded (smallest
// failing index; knn_stage's query error first, as the stages run).
void raise_pass_failures(const FailFlags& fails) {
    if (fails.h[kFailQuery] != LLONG_MAX)
        throw Failure(AIDW_ERR_RUNTIME,
                      "knn_stage: query " + std::to_string(fails.h[kFailQuery]) +
                          ": locate_cell: point lies outside the covered region",
                      fails.h[kFailQuery]);
    if (fails.h[kFailData] != LLONG_MAX)
        throw Failure(AIDW_ERR_DOMAIN, "locate_cell: data point " + std::to_string(fails.h[kFailData]) +
                                           " lies outside the covered region",
                      fails.h[kFailData]);
    if (fails.h[kFailAlpha] != LLONG_MAX)
        throw Failure(AIDW_ERR_RUNTIME,
                      "aidw_predict_all: query " + std::to_string(fails.h[kFailAlpha]) +
                          ": alpha_from_mu: mu outside [0, 1]",
                      fails.h[kFailAlpha]);
}

// cmd_raster's query lattice (cli.hpp:496-507) generated in HBM: row-major,
// northernmost row first, rows [row0, row0 + rows) of the ny-row lattice.
// Explicit round-to-nearest ops keep the reference's two-rounding form.
__global__ void lattice_kernel(size_t nx, size_t ny, double min_x, double min_y, double sx,
                               double sy, size_t row0, size_t rows, double* __restrict__ qx,
                               double* __restrict__ qy) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nx * rows) return;
    const size_t r = row0 + i / nx, c = i % nx;
    qx[i] = __dadd_rn(min_x, __dmul_rn(__dadd_rn(static_cast<double>(c), 0.5), sx));
    qy[i] = __dadd_rn(min_y, __dmul_rn(__dadd_rn(static_cast<double>(ny - 1 - r), 0.5), sy));
}

void lattice_device(size_t nx, size_t ny, const double* bbox, size_t row0, size_t rows,
                    double* d_qx, double* d_qy, cudaStream_t s) {
    if (nx < 1 || ny < 1)
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "cmd_raster: nx and ny must be >= 1");
    if (row0 + rows > ny) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "cmd_raster: row range outside the lattice");
    const double sx = (bbox[2] - bbox[0]) / static_cast<double>(nx);  // cli.hpp:496-497
    const double sy = (bbox[3] - bbox[1]) / static_cast<double>(ny);
    if (nx * rows)
        LAUNCH(lattice_kernel, ceil_div(nx * rows, kThreads), kThreads, 0, s, nx, ny, bbox[0],
               bbox[1], sx, sy, row0, rows, d_qx, d_qy);
}

// Per-call workspace (see DBuf): a cached device buffer per device, sized
// by the largest call so far (plus what overflowed), handed to one call at
// a time.  Recycled after the call's stream is synchronised.
struct ArenaCache {
    std::mutex mu;
    std::vector<Arena> free_list;
};
ArenaCache g_arena_cache[64];

struct ArenaScope {
    Arena a;
    Arena* prev = nullptr;
    int dev = 0;
    explicit ArenaScope(cudaStream_t s) {
        CK(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lock(g_arena_cache[dev & 63].mu);
            auto& fl = g_arena_cache[dev & 63].free_list;
            if (!fl.empty()) {
                a = fl.back();
                fl.pop_back();
            }
        }
        a.used = a.overflow = 0;
        a.stream = s;
        prev = t_arena;
        t_arena = &a;
    }
    ~ArenaScope() {
        t_arena = prev;
        // normally a no-op (the call synchronised); on an exception path it
        // keeps in-flight kernels off a recycled workspace
        if (cudaStreamSynchronize(a.stream) != cudaSuccess) cudaGetLastError();
        // much larger than the last few calls needed (> 256 MiB, 8x their
        // use, 3 calls in a row): give it back, the next call re-sizes it
        a.small = (a.cap > (size_t(256) << 20) && (a.used + a.overflow) * 8 < a.cap) ? a.small + 1 : 0;
        if (a.small >= 3 && !a.overflow) {
            cudaFreeAsync(a.base, a.stream);
            if (cudaStreamSynchronize(a.stream) != cudaSuccess) cudaGetLastError();
            a.base = nullptr;
            a.cap = 0;
            a.small = 0;
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
                cudaMemPoolTrimTo(pool, g_pool_keep[dev & 63]);
        }
        if (a.overflow) {  // grow for the next call, from the warm pool
            if (a.base) cudaFreeAsync(a.base, a.stream);
            a.base = nullptr;
            a.cap = 0;
            const size_t want = ((a.used + a.overflow) * 5 / 4 + (size_t(1) << 20)) & ~size_t(255);
            if (cudaMallocAsync(reinterpret_cast<void**>(&a.base), want, a.stream) == cudaSuccess &&
                cudaStreamSynchronize(a.stream) == cudaSuccess)
                a.cap = want;
            else
                cudaGetLastError();
        }
        a.used = a.overflow = 0;
        a.stream = nullptr;
        std::lock_guard<std::mutex> lock(g_arena_cache[dev & 63].mu);
        g_arena_cache[dev & 63].free_list.push_back(a);
    }
    ArenaScope(const ArenaScope&) = delete;
    ArenaScope& operator=(const ArenaScope&) = delete;
};

// ---- CUDA-graph cache of fused passes.  A pass whose plan, buffers and
// workspace are those of an earlier pass is the same launch sequence, so it
// is captured once (on its second occurrence: the first run sized the
// workspace) and replayed with one cudaGraphLaunch — ~40 kernel launches of
// host overhead become one, which is most of a 10K x 10K pass.  The key
// holds every host value a kernel of the pass receives: the plan (bbox, value
// hull, grid, k, alpha parameters), the run config, the device buffers, the
// workspace base / offset, the device and the process-wide weighting knobs.
struct GraphKeyPod {
    int dev, precision, recipe;
    size_t m, n, slab, arena_cap, arena_used;
    const void* ptr[8];
    aidw_run_config cfg;
    double ext[6];
};

struct GraphEntry {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec = nullptr;
    PassEvents ev;
    size_t used_after = 0;  // workspace offset after the captured pass
    long long kernels = 0;  // kernel nodes (counted as launches on replay)
    long long uses = 0;
};

std::mutex g_graph_mu;
std::vector<std::unique_ptr<GraphEntry>> g_graphs;      // most recent last, <= kMaxGraphs
std::vector<std::vector<unsigned char>> g_graph_seen;    // keys run once without overflow
constexpr size_t kMaxGraphs = 16;
std::atomic<int> g_graphs_enabled{[] {
    const char* e = std::getenv("AIDW_GRAPHS");
    return (e && e[0] == '0') ? 0 : 1;
}()};
std::atomic<long long> g_graph_replays{0}, g_graph_captures{0};

std::vector<unsigned char> graph_key(const PipelineIO& io, const aidw_run_config& cfg,
                                     const PassPlan& pl, const Arena* arena, cudaStream_t s) {
    GraphKeyPod k;
    std::memset(&k, 0, sizeof k);
    CK(cudaGetDevice(&k.dev));
    k.precision = g_precision.load();
    k.recipe = alpha4_recipe_enabled() ? 1 : 0;
    k.m = io.m;
    k.n = io.n;
    k.slab = query_slab(weight_split(io.m).chunks);
    k.arena_cap = arena->cap;
    k.arena_used = arena->used;
    const void* p[8] = {io.dx, io.dy, io.dz, io.qx, io.qy, io.pred, io.alpha, arena->base};
    std::memcpy(k.ptr, p, sizeof p);
    k.cfg = cfg;
    const double e[6] = {pl.ext.box.min_x, pl.ext.box.min_y, pl.ext.box.max_x, pl.ext.box.max_y,
                         pl.hull_in_pass ? 1.0 : 0.0, 0.0};
    std::memcpy(k.ext, e, sizeof e);
    (void)s;
    std::vector<unsigned char> out(sizeof k);
    std::memcpy(out.data(), &k, sizeof k);
    return out;
}

// Runs the pass's device work: a cached graph, a fresh capture, or eagerly.
// Returns the events that time it.
const PassEvents& run_pass(const PassPlan& pl, const PipelineIO& io, const aidw_run_config& cfg,
                           FailFlags& fails, PassEvents& eager_ev, Arena* arena, cudaStream_t s) {
    const bool graphable = g_graphs_enabled.load() && arena && arena->stream == s && arena->base;
    std::vector<unsigned char> key;
    if (graphable) {
        key = graph_key(io, cfg, pl, arena, s);
        std::unique_lock<std::mutex> lk(g_graph_mu);
        for (size_t i = 0; i < g_graphs.size(); ++i) {
            if (g_graphs[i]->key == key) {
                GraphEntry* e = g_graphs[i].get();
                std::rotate(g_graphs.begin() + i, g_graphs.begin() + i + 1, g_graphs.end());
                lk.unlock();
                // the workspace holds the same buffers at the same offsets:
                // advance it as the captured pass did
                arena->used = e->used_after;
                CK(cudaGraphLaunch(e->exec, s));
                g_launches.fetch_add(e->kernels, std::memory_order_relaxed);
                ++e->uses;
                g_graph_replays.fetch_add(1);
                return e->ev;
            }
        }
        const bool seen = std::find(g_graph_seen.begin(), g_graph_seen.end(), key) != g_graph_seen.end();
        lk.unlock();
        if (seen) {  // second occurrence: capture, keep, replay
            auto e = std::make_unique<GraphEntry>();
            e->key = key;
            e->ev.create();
            const size_t used0 = arena->used, over0 = arena->overflow;
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            bool ok = true;
            t_launch_sink = &e->kernels;
            try {
                fails.init(s);
                enqueue_pass(pl, io, cfg, e->ev, fails, s);
            } catch (...) {
                ok = false;
            }
            t_launch_sink = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(s, &graph);
            ok = ok && ce == cudaSuccess && arena->overflow == over0;
            if (ok && cudaGraphInstantiate(&e->exec, graph, 0) != cudaSuccess) ok = false;
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            if (ok) {
                e->used_after = arena->used;
                CK(cudaGraphLaunch(e->exec, s));
                g_launches.fetch_add(e->kernels);
                g_graph_captures.fetch_add(1);
                const PassEvents* ev = &e->ev;
                std::lock_guard<std::mutex> g(g_graph_mu);
                g_graphs.push_back(std::move(e));
                if (g_graphs.size() > kMaxGraphs) {
                    GraphEntry* old = g_graphs.front().get();
                    cudaStreamSynchronize(s);
                    cudaGraphExecDestroy(old->exec);
                    old->ev.destroy();
                    g_graphs.erase(g_graphs.begin());
                }
                return *ev;
            }
            // capture failed (e.g. the workspace overflowed inside it): run eagerly
            if (e->exec) cudaGraphExecDestroy(e->exec);
            e->ev.destroy();
            arena->used = used0;
            arena->overflow = over0;
        }
    }
    eager_ev.create();
    fails.init(s);
    enqueue_pass(pl, io, cfg, eager_ev, fails, s);
    if (graphable && arena->overflow == 0) {
        std::lock_guard<std::mutex> g(g_graph_mu);
        if (std::find(g_graph_seen.begin(), g_graph_seen.end(), key) == g_graph_seen.end()) {
            g_graph_seen.push_back(key);
            if (g_graph_seen.size() > 4 * kMaxGraphs) g_graph_seen.erase(g_graph_seen.begin());
        }
    }
    return eager_ev;
}

// A workspace for the call unless the caller (e.g. aidw_run_pipeline, whose
// uploads live in it too) already opened one on this stream.
struct MaybeArena {
    std::unique_ptr<ArenaScope> own;
    explicit MaybeArena(cudaStream_t s) {
        if (!(t_arena && t_arena->stream == s)) own = std::make_unique<ArenaScope>(s);
    }
};

void pipeline_entry(const PipelineIO& io, const aidw_run_config& cfg, aidw_run_stats* st,
                    cudaStream_t s, double h2d_ms, const std::chrono::steady_clock::time_point& t0,
                    double* h_pred, double* h_alpha) {
    const long long launches0 = g_launches.load();
    const auto ta = std::chrono::steady_clock::now();
    MaybeArena arena(s);  // declared first: destroyed after every DBuf of the call
    const auto tb = std::chrono::steady_clock::now();
    aidw_run_stats local{};
    DBuf<double> hull(6, s);
    const auto tp0 = std::chrono::steady_clock::now();
    const PassPlan pl = plan_pass(io, cfg, &local, hull.get(), s);
    const auto tp1 = std::chrono::steady_clock::now();
    FailFlags fails(s, /*defer_init=*/true);
    PassEvents eager;
    struct EventsGuard {
        PassEvents& e;
        ~EventsGuard() { e.destroy(); }
    } guard{eager};
    const PassEvents& ev = run_pass(pl, io, cfg, fails, eager, t_arena, s);
    const auto tp2 = std::chrono::steady_clock::now();
    double d2h_ms = 0.0;
    const auto c0 = std::chrono::steady_clock::now();
    if (h_pred) {  // results and the failure flags come back behind one synchronisation
        d2h(h_pred, io.pred, io.n, s);
        if (h_alpha) d2h(h_alpha, io.alpha, io.n, s);
    }
    fails.fetch(s);  // failure indices and pass counters, one copy
    if (h_pred)
        d2h_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
    if (host_trace()) {
        const auto tp3 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "[aidw pass] m %zu n %zu: entry %.1f, arena %.1f, hull %.1f, plan %.1f, "
                     "enqueue %.1f, wait+fetch %.1f us\n", io.m, io.n, us(t0, ta), us(ta, tb),
                     us(tb, tp0), us(tp0, tp1), us(tp1, tp2), us(tp2, tp3));
    }
    raise_pass_failures(fails);
    if (st) {
        *st = local;
        // idw mode has no build / kNN stage (cli.hpp:227-234): exactly 0 ms
        const bool idw = cfg.mode == AIDW_MODE_IDW;
        st->build_ms = idw ? 0.0 : Events::ms(ev.build0, ev.build1);
        st->knn_ms = idw ? 0.0 : Events::ms(ev.build1, ev.knn1);
        st->interp_ms = Events::ms(ev.knn1, ev.interp1);
        st->weight_kernel_ms = Events::ms(ev.k4b, ev.k4e);
        st->knn_kernel_ms = idw ? 0.0 : Events::ms(ev.knnb, ev.knne);
        st->h2d_ms = h2d_ms;
        st->d2h_ms = d2h_ms;
        st->worker_count = cfg.workers > 0 ? cfg.workers : 1;
        st->pairs = static_cast<int64_t>(io.m) * static_cast<int64_t>(io.n);
        st->alpha4_queries = fails.h[kCountAlpha4];
        st->knn_candidates = fails.h[kCountCand];
        st->knn_ref_candidates = fails.h[kCountRefCand];
        st->kernel_launches = g_launches.load() - launches0;
        st->total_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
}

// ------------------------------------------------------------ multi-device
// SURVEY §8e's single-process model: one host thread per device, the data
// replicated to every device, a contiguous slice of the queries (or of the
// raster's lattice rows) per device, and the global bbox(data ∪ all
// queries) combined on the host before any grid is built — so every device
// builds the identical grid, area and snap tolerance, and the result is
// bit-identical to a one-device run (per-query formulas and summation order
// depend on the query and m only).  Device list: aidw_set_devices or
// AIDW_DEVICES="0,1,..."; a list may repeat a device (shards then share it).
std::mutex g_dev_mu;
std::vector<int> g_devices;
bool g_dev_env_read = false;

std::vector<int> device_list() {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_dev_env_read) {
        g_dev_env_read = true;
        if (const char* v = std::getenv("AIDW_DEVICES")) {
            std::vector<int> ids;
            const char* p = v;
            while (*p) {
                char* end = nullptr;
                const long id = std::strtol(p, &end, 10);
                if (end == p) break;
                ids.push_back(static_cast<int>(id));
                p = *end == ',' ? end + 1 : end;
            }
            if (g_devices.empty()) g_devices = ids;
        }
    }
    return g_devices;
}

// One shard's device buffers (released on the shard's own thread); the
// data arrays are its device's replica (shared by the shards on a device).
struct ShardBufs {
    const double *dx = nullptr, *dy = nullptr, *dz = nullptr;
    DBuf<double> qx, qy, pred, alpha;
    double h2d_ms = 0.0;
    void release() {
        qx.release(), qy.release();
        pred.release(), alpha.release();
    }
};

// The data set on every listed device: one H2D to the first, ncclBroadcast
// to the others (replicate.cu); each shard points at its device's replica.
double replicate_for_shards(const std::vector<int>& devs, const double* dx, const double* dy,
                            const double* dz, size_t m, Replicas& reps, ShardBufs* b) {
    const auto c0 = std::chrono::steady_clock::now();
    replicate_data(devs, dx, dy, dz, m, reps);
    for (size_t d = 0; d < devs.size(); ++d) {
        const int r = reps.slot_of(devs[d]);
        b[d].dx = reps.x[r];
        b[d].dy = reps.y[r];
        b[d].dz = reps.z[r];
    }
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
}

// A reusable-free count-down barrier for the shard threads.
struct ShardBarrier {
    std::mutex mu;
    std::condition_variable cv;
    size_t left;
    explicit ShardBarrier(size_t n) : left(n) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (--left == 0) {
            cv.notify_all();
        } else {
            cv.wait(lk, [this] { return left == 0; });
        }
    }
};

void shard_bounds(size_t n, size_t parts, size_t k, size_t& lo, size_t& hi) {
    const size_t base = n / parts, extra = n % parts;
    lo = k * base + std::min(k, extra);
    hi = lo + base + (k < extra ? 1 : 0);
}

void merge_stats(aidw_run_stats& out, const aidw_run_stats* st, size_t count) {
    out = st[0];
    for (size_t d = 1; d < count; ++d) {
        const aidw_run_stats& t = st[d];
        out.build_ms = std::max(out.build_ms, t.build_ms);
        out.knn_ms = std::max(out.knn_ms, t.knn_ms);
        out.interp_ms = std::max(out.interp_ms, t.interp_ms);
        out.total_ms = std::max(out.total_ms, t.total_ms);
        out.weight_kernel_ms = std::max(out.weight_kernel_ms, t.weight_kernel_ms);
        out.knn_kernel_ms = std::max(out.knn_kernel_ms, t.knn_kernel_ms);
        out.h2d_ms = std::max(out.h2d_ms, t.h2d_ms);
        out.d2h_ms = std::max(out.d2h_ms, t.d2h_ms);
        out.pairs += t.pairs;
        out.alpha4_queries += t.alpha4_queries;
        out.knn_candidates += t.knn_candidates;
        out.knn_ref_candidates += t.knn_ref_candidates;
        out.kernel_launches += t.kernel_launches;
    }
}

// One shard's work: `prep` uploads / generates its inputs on the shard's
// device and returns its partial bbox; then (after all shards met) `run`
// gets the global box.  Returns false if any shard failed (the caller then
// re-runs on one device, which raises the reference's exact error).
using ShardPrep = std::function<Box(size_t, cudaStream_t)>;
using ShardRun = std::function<void(size_t, cudaStream_t, const Box&)>;
using ShardFinish = std::function<void(size_t)>;

void shard_thread(size_t d, int dev, const ShardPrep& prep, const ShardRun& run,
                  const ShardFinish& finish, Box* boxes, char* failed, size_t D,
                  ShardBarrier* sync) {
    cudaStream_t s = nullptr;
    try {
        CK(cudaSetDevice(dev));
        current_device();  // pool set-up for this device
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        boxes[d] = prep(d, s);
    } catch (...) {
        failed[d] = 1;
    }
    sync->arrive_and_wait();
    bool any = false;
    for (size_t k = 0; k < D; ++k) any |= failed[k] != 0;
    if (!any) {
        Box g = boxes[0];
        for (size_t k = 1; k < D; ++k) {
            g.min_x = std::min(g.min_x, boxes[k].min_x);
            g.min_y = std::min(g.min_y, boxes[k].min_y);
            g.max_x = std::max(g.max_x, boxes[k].max_x);
            g.max_y = std::max(g.max_y, boxes[k].max_y);
        }
        try {
            run(d, s, g);
        } catch (...) {
            failed[d] = 1;
        }
    }
    try {
        finish(d);  // buffers go back on this device / stream
    } catch (...) {
    }
    if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
}

// One shard's work: `prep` uploads / generates its inputs on the shard's
// device and returns its partial bbox; then (after all shards met) `run`
// gets the global box; `finish` releases its buffers.  Returns false if any
// shard failed (the caller then re-runs on one device, which raises the
// reference's exact error).
bool run_sharded(const std::vector<int>& devs, const ShardPrep& prep, const ShardRun& run,
                 const ShardFinish& finish) {
    const size_t D = devs.size();
    std::unique_ptr<Box[]> boxes(new Box[D]);
    std::unique_ptr<char[]> failed(new char[D]());
    ShardBarrier sync(D);
    std::unique_ptr<std::thread[]> pool(new std::thread[D]);
    for (size_t d = 0; d < D; ++d)
        pool[d] = std::thread(shard_thread, d, devs[d], std::cref(prep), std::cref(run),
                              std::cref(finish), boxes.get(), failed.get(), D, &sync);
    for (size_t d = 0; d < D; ++d) pool[d].join();
    for (size_t d = 0; d < D; ++d)
        if (failed[d]) return false;
    return true;
}

// run_pipeline over query shards, one per listed device.
struct PipelineShards {
    const double *dx, *dy, *dz, *qx, *qy;
    size_t m, n, D;
    aidw_run_config cfg;
    double *pred_out, *alpha_out;
    std::chrono::steady_clock::time_point t0;
    ShardBufs* b;
    aidw_run_stats* st;

    Box prep(size_t d, cudaStream_t s) {
        size_t lo, hi;
        shard_bounds(n, D, d, lo, hi);
        const auto c0 = std::chrono::steady_clock::now();
        h2d(b[d].qx, qx + lo, hi - lo, s);
        h2d(b[d].qy, qy + lo, hi - lo, s);
        b[d].pred.alloc(hi - lo, s);
        b[d].alpha.alloc(hi - lo, s);
        const Box e = extents_box(b[d].dx, b[d].dy, m, b[d].qx.get(), b[d].qy.get(), hi - lo, s);
        b[d].h2d_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
        return e;
    }
    void run(size_t d, cudaStream_t s, const Box& g) {
        size_t lo, hi;
        shard_bounds(n, D, d, lo, hi);
        aidw_run_config c = cfg;
        if (!c.use_bbox) {
            c.use_bbox = 1;
            c.bbox[0] = g.min_x;
            c.bbox[1] = g.min_y;
            c.bbox[2] = g.max_x;
            c.bbox[3] = g.max_y;
        }
        PipelineIO io{b[d].dx, b[d].dy, b[d].dz, b[d].qx.get(), b[d].qy.get(),
                      m, hi - lo, b[d].pred.get(), b[d].alpha.get()};
        pipeline_entry(io, c, &st[d], s, b[d].h2d_ms, t0, pred_out + lo,
                       alpha_out ? alpha_out + lo : nullptr);
    }
};

bool pipeline_multi(const std::vector<int>& devs, const double* dx, const double* dy,
                    const double* dz, size_t m, const double* qx, const double* qy, size_t n,
                    const aidw_run_config& cfg, double* pred_out, double* alpha_out,
                    aidw_run_stats* stats, std::chrono::steady_clock::time_point t0) {
    const size_t D = devs.size();
    std::unique_ptr<ShardBufs[]> bufs(new ShardBufs[D]);
    std::unique_ptr<aidw_run_stats[]> st(new aidw_run_stats[D]());
    Replicas reps;
    const double rep_ms = replicate_for_shards(devs, dx, dy, dz, m, reps, bufs.get());
    for (size_t d = 0; d < D; ++d) bufs[d].h2d_ms = rep_ms;
    PipelineShards job{dx, dy, dz, qx, qy, m, n, D, cfg, pred_out, alpha_out, t0, bufs.get(), st.get()};
    PipelineShards* j = &job;
    ShardBufs* b = bufs.get();
    const bool ok = run_sharded(
        devs, [j](size_t d, cudaStream_t s) { return j->prep(d, s); },
        [j](size_t d, cudaStream_t s, const Box& g) { j->run(d, s, g); },
        [b](size_t d) { b[d].release(); });
    if (ok && stats) merge_stats(*stats, st.get(), D);
    return ok;
}

// run_raster over lattice-row shards, one per listed device.
struct RasterShards {
    const double *dx, *dy, *dz;
    size_t m, nx, ny, D;
    aidw_run_config cfg;
    double *raster_out, *alpha_out;
    std::chrono::steady_clock::time_point t0;
    ShardBufs* b;
    aidw_run_stats* st;

    Box prep(size_t d, cudaStream_t s) {
        return extents_box(b[d].dx, b[d].dy, m, nullptr, nullptr, 0, s);
    }
    void run(size_t d, cudaStream_t s, const Box& g) {
        size_t r0, r1;
        shard_bounds(ny, D, d, r0, r1);
        const size_t n = nx * (r1 - r0);
        const double bb[4] = {g.min_x, g.min_y, g.max_x, g.max_y};
        b[d].qx.alloc(n, s);
        b[d].qy.alloc(n, s);
        b[d].pred.alloc(n, s);
        b[d].alpha.alloc(n, s);
        lattice_device(nx, ny, bb, r0, r1 - r0, b[d].qx.get(), b[d].qy.get(), s);
        aidw_run_config c = cfg;
        c.use_bbox = 1;
        std::memcpy(c.bbox, bb, sizeof bb);
        PipelineIO io{b[d].dx, b[d].dy, b[d].dz, b[d].qx.get(), b[d].qy.get(),
                      m, n, b[d].pred.get(), b[d].alpha.get()};
        pipeline_entry(io, c, &st[d], s, b[d].h2d_ms, t0, raster_out + nx * r0,
                       alpha_out ? alpha_out + nx * r0 : nullptr);
    }
};

bool raster_multi(const std::vector<int>& devs, const double* dx, const double* dy,
                  const double* dz, size_t m, size_t nx, size_t ny, const aidw_run_config& cfg,
                  double* raster_out, double* alpha_out, double* bbox_out, aidw_run_stats* stats,
                  std::chrono::steady_clock::time_point t0) {
    const size_t D = devs.size();
    std::unique_ptr<ShardBufs[]> bufs(new ShardBufs[D]);
    std::unique_ptr<aidw_run_stats[]> st(new aidw_run_stats[D]());
    std::unique_ptr<Box[]> box(new Box[1]);
    Replicas reps;
    const double rep_ms = replicate_for_shards(devs, dx, dy, dz, m, reps, bufs.get());
    for (size_t d = 0; d < D; ++d) bufs[d].h2d_ms = rep_ms;
    RasterShards job{dx, dy, dz, m, nx, ny, D, cfg, raster_out, alpha_out, t0, bufs.get(), st.get()};
    RasterShards* j = &job;
    ShardBufs* b = bufs.get();
    Box* kept = box.get();
    const bool ok = run_sharded(
        devs, [j](size_t d, cudaStream_t s) { return j->prep(d, s); },
        [j, kept](size_t d, cudaStream_t s, const Box& g) {
            if (d == 0) *kept = g;
            j->run(d, s, g);
        },
        [b](size_t d) { b[d].release(); });
    if (ok) {
        if (stats) merge_stats(*stats, st.get(), D);
        if (bbox_out) {
            bbox_out[0] = kept->min_x;
            bbox_out[1] = kept->min_y;
            bbox_out[2] = kept->max_x;
            bbox_out[3] = kept->max_y;
        }
    }
    return ok;
}

// build_index's argument checks (grid.hpp:178-183).
void build_index_checks(size_t m, const aidw_grid_config* cfg) {
    if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "build_index: data set is empty");
    if (m > static_cast<size_t>(std::numeric_limits<uint32_t>::max()) - 1)
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "build_index: too many points for 32-bit ids");
    if (!cfg || cfg->n_col < 1 || cfg->n_row < 1 || !(cfg->cell_width > 0.0))
        throw Failure(AIDW_ERR_INVALID_ARGUMENT, "build_index: invalid grid configuration");
}

// knn_stage's k_eff / exhausted and per-query preconditions (knn.hpp:255-271,
// grid_knn :212-223, brute_force_knn :100-108): the errors every query would
// raise are reported for query 0, the smallest index.
int knn_stage_prologue(size_t n, size_t m, int32_t k, bool grid, int32_t* k_eff_out,
                       int32_t* exhausted_out) {
    const int k_eff = grid ? static_cast<int>(std::min<int64_t>(k, static_cast<int64_t>(m))) : k;
    const bool exhausted = grid && static_cast<int64_t>(m) < k;
    if (k_eff_out) *k_eff_out = k_eff;
    if (exhausted_out) *exhausted_out = exhausted ? 1 : 0;
    if (n == 0) return k_eff;
    if (grid) {
        if (m == 0) throw Failure(AIDW_ERR_RUNTIME, "knn_stage: query 0: grid_knn: index holds no points", 0);
        if (k < 1) throw Failure(AIDW_ERR_RUNTIME, "knn_stage: query 0: grid_knn: k must be >= 1", 0);
    } else {
        if (m == 0)
            throw Failure(AIDW_ERR_RUNTIME, "knn_stage: query 0: brute_force_knn: data set is empty", 0);
        if (k < 1 || static_cast<size_t>(k) > m)
            throw Failure(AIDW_ERR_RUNTIME,
                          "knn_stage: query 0: brute_force_knn: k = " + std::to_string(k) +
                              " outside [1, " + std::to_string(m) + "]", 0);
    }
    return k_eff;
}

// The grid engine of knn_stage over device CSR arrays: queries uploaded,
// sorted by cell (locate failures -> the smallest failing query), K2, and
// the flat outputs copied back to the caller's buffers.
void knn_grid_stage(const double* qx, const double* qy, size_t n, const aidw_grid_config& cfg,
                    const uint32_t* d_cs, const uint32_t* d_ids, const double2* d_xy, size_t m,
                    int k, int k_eff, double* d2_out, uint32_t* idx_out, double* avg_out,
                    cudaStream_t s) {
    FailFlags fails(s);
    DBuf<double> dqx, dqy, d2(n * static_cast<size_t>(k_eff), s), avg(n, s);
    DBuf<uint32_t> ids(idx_out ? n * static_cast<size_t>(k_eff) : 0, s), perm, qcell;
    h2d(dqx, qx, n, s);
    h2d(dqy, qy, n, s);
    const GridGeom geom = make_geom(cfg);
    const int nbc = sort_queries_by_cell(dqx.get(), dqy.get(), n, geom, perm, qcell, fails.slot(kFailQuery), s);
    KnnArgs a;
    a.qx = dqx.get();
    a.qy = dqy.get();
    a.n = n;
    a.m = m;
    a.k = k;
    a.k_eff = k_eff;
    a.d2_out = d2.get();
    a.id_out = idx_out ? ids.get() : nullptr;
    a.avg_out = avg.get();
    a.g = geom;
    a.cell_start = d_cs;
    a.sorted_ids = d_ids;
    a.sorted_xy = d_xy;
    a.perm = perm.get();
    a.qcell = qcell.get();
    a.qkey_nbc = nbc;
    // a query outside the grid makes K2 skip it (locate fails the same way
    // in both kernels); the error is raised after the single synchronisation
    run_knn_grid(a, s);
    d2h(d2_out, d2.get(), n * static_cast<size_t>(k_eff), s);
    if (idx_out) d2h(idx_out, ids.get(), n * static_cast<size_t>(k_eff), s);
    d2h(avg_out, avg.get(), n, s);
    fails.fetch(s);
    if (fails.h[kFailQuery] != LLONG_MAX) {
        const long long i = fails.h[kFailQuery];
        throw Failure(AIDW_ERR_RUNTIME,
                      "knn_stage: query " + std::to_string(i) + ": " + locate_msg(qx[i], qy[i]), i);
    }
}

// Page-locked staging cache (aidw_pinned_alloc): freed blocks are kept (up
// to 2 GiB) and reused for requests they cover without wasting over half.
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;
std::map<void*, size_t> g_pin_size;
size_t g_pin_cached = 0;

void* pinned_alloc(size_t bytes) {
    if (bytes == 0) bytes = 1;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.lower_bound(bytes);  // the smallest cached block that fits
        if (it != g_pin_free.end()) {
            void* p = it->second;
            g_pin_cached -= it->first;
            g_pin_free.erase(it);
            return p;
        }
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return nullptr;
    }
    // at least 64 MiB: pinning costs ~1 ms per 4 MiB, paid once per block
    const size_t size =
        std::max<size_t>((bytes + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1), size_t(64) << 20);
    void* p = nullptr;
    if (cudaHostAlloc(&p, size, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_size[p] = size;
    return p;
}

void pinned_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_size.find(p);
    if (it == g_pin_size.end()) return;
    const size_t size = it->second;
    if (g_pin_cached + size > (size_t(2) << 30)) {
        g_pin_size.erase(it);
        cudaFreeHost(p);
        return;
    }
    g_pin_free.emplace(size, p);
    g_pin_cached += size;
}

// Makes `dev` current for a scope (mirror handles belong to one device).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace
}  // namespace aidwb

using namespace aidwb;

// The device mirror behind aidw_index* (include/aidw_capi.h): the grid's CSR
// arrays resident on device `dev`, allocated and released on its own stream.
struct aidw_index {
    int dev = 0;
    aidw_grid_config cfg{};
    size_t m = 0;
    cudaStream_t s = nullptr;
    DeviceGrid g;
    ~aidw_index() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
        g.cell_start.release();  // back to the pool, on s
        g.sorted_ids.release();
        g.sorted_x.release();
        g.sorted_y.release();
        g.sorted_xy.release();
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
        if (prev >= 0) cudaSetDevice(prev);
        cudaGetLastError();
    }
};

extern "C" {

int aidw_capi_version(void) { return AIDW_CAPI_VERSION; }

int64_t aidw_kernel_launch_count(void) { return g_launches.load(); }

void aidw_set_weight_precision(int32_t precision) {
    g_precision.store(precision == AIDW_PRECISION_FP64 ? AIDW_PRECISION_FP64 : AIDW_PRECISION_FP32);
}

int32_t aidw_get_weight_precision(void) { return g_precision.load(); }

void aidw_set_alpha4_recipe(int32_t enabled) { set_alpha4_recipe(enabled != 0); }

int32_t aidw_weight_engine(int64_t m) {
    return weight_tc_selected(weight_split(m > 0 ? static_cast<size_t>(m) : 0)) ? 1 : 0;
}

void aidw_set_query_slab(int64_t queries) { set_query_slab(queries > 0 ? static_cast<size_t>(queries) : 0); }

int aidw_device_info(char* name, size_t cap, int32_t* sm_count, aidw_error* err) {
    return guarded(err, [&] {
        const int dev = current_device();
        cudaDeviceProp p;
        CK(cudaGetDeviceProperties(&p, dev));
        if (name && cap) {
            std::strncpy(name, p.name, cap - 1);
            name[cap - 1] = '\0';
        }
        if (sm_count) *sm_count = p.multiProcessorCount;
    });
}

int aidw_build_index(const double* xs, const double* ys, size_t m, const aidw_grid_config* cfg,
                     uint32_t* sorted_ids, uint32_t* cell_start, double* sorted_x,
                     double* sorted_y, aidw_error* err) {
    return guarded(err, [&] {
        build_index_checks(m, cfg);
        StreamScope ss;
        cudaStream_t s = ss.s;
        FailFlags fails(s);
        DBuf<double> dx, dy;
        h2d(dx, xs, m, s);
        h2d(dy, ys, m, s);
        DeviceGrid g;
        build_grid_device(dx.get(), dy.get(), m, *cfg, g, fails.slot(kFailData), s, true);
        fails.fetch(s);
        if (fails.h[kFailData] != LLONG_MAX) {
            const long long i = fails.h[kFailData];
            throw Failure(AIDW_ERR_DOMAIN, locate_msg(xs[i], ys[i]), i);
        }
        d2h(sorted_ids, g.sorted_ids.get(), m, s);
        d2h(cell_start, g.cell_start.get(), g.cells + 1, s);
        d2h(sorted_x, g.sorted_x.get(), m, s);
        d2h(sorted_y, g.sorted_y.get(), m, s);
        ss.sync();
    });
}

int aidw_knn_stage(const double* qx, const double* qy, size_t n, const aidw_grid_config* cfg,
                   const uint32_t* cell_start, const uint32_t* sorted_ids,
                   const double* sorted_x, const double* sorted_y, const double* dx,
                   const double* dy, size_t m, int32_t k, int32_t engine, double* d2_out,
                   uint32_t* idx_out, double* avg_out, int32_t* k_eff_out,
                   int32_t* exhausted_out, aidw_error* err) {
    return guarded(err, [&] {
        const bool grid = engine == AIDW_ENGINE_GRID;
        if (grid && (!cfg || !cell_start || (m > 0 && (!sorted_ids || !sorted_x || !sorted_y))))
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "knn_stage: grid engine requires a grid index");
        const int k_eff = knn_stage_prologue(n, m, k, grid, k_eff_out, exhausted_out);
        if (n == 0) return;
        StreamScope ss;
        cudaStream_t s = ss.s;
        if (grid) {
            const size_t cells = static_cast<size_t>(cfg->n_col) * static_cast<size_t>(cfg->n_row);
            DBuf<double> sx, sy;
            DBuf<double2> sxy;
            DBuf<uint32_t> cs, sid;
            h2d(cs, cell_start, cells + 1, s);
            h2d(sid, sorted_ids, m, s);
            h2d(sx, sorted_x, m, s);
            h2d(sy, sorted_y, m, s);
            sxy.alloc(m, s);
            interleave_xy(sx.get(), sy.get(), m, sxy.get(), s);
            knn_grid_stage(qx, qy, n, *cfg, cs.get(), sid.get(), sxy.get(), m, k, k_eff, d2_out,
                           idx_out, avg_out, s);
        } else {
            FailFlags fails(s);
            DBuf<double> dqx, dqy, d2(n * static_cast<size_t>(k_eff), s), avg(n, s);
            DBuf<uint32_t> ids(idx_out ? n * static_cast<size_t>(k_eff) : 0, s);
            DBuf<double> ddx, ddy;
            h2d(dqx, qx, n, s);
            h2d(dqy, qy, n, s);
            h2d(ddx, dx, m, s);
            h2d(ddy, dy, m, s);
            KnnArgs a;
            a.qx = dqx.get();
            a.qy = dqy.get();
            a.n = n;
            a.m = m;
            a.k = k;
            a.k_eff = k_eff;
            a.d2_out = d2.get();
            a.id_out = idx_out ? ids.get() : nullptr;
            a.avg_out = avg.get();
            a.dx = ddx.get();
            a.dy = ddy.get();
            run_knn_brute(a, s);
            d2h(d2_out, d2.get(), n * static_cast<size_t>(k_eff), s);
            if (idx_out) d2h(idx_out, ids.get(), n * static_cast<size_t>(k_eff), s);
            d2h(avg_out, avg.get(), n, s);
        }
        ss.sync();
    });
}

int aidw_build_index_mirror(const double* xs, const double* ys, size_t m,
                            const aidw_grid_config* cfg, uint32_t* sorted_ids,
                            uint32_t* cell_start, double* sorted_x, double* sorted_y,
                            aidw_index** mirror, aidw_error* err) {
    if (mirror) *mirror = nullptr;
    return guarded(err, [&] {
        build_index_checks(m, cfg);
        auto h = std::make_unique<aidw_index>();
        h->dev = current_device();
        h->cfg = *cfg;
        h->m = m;
        CK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
        cudaStream_t s = h->s;
        {
            FailFlags fails(s);
            DBuf<double> dx, dy;
            h2d(dx, xs, m, s);
            h2d(dy, ys, m, s);
            build_grid_device(dx.get(), dy.get(), m, *cfg, h->g, fails.slot(kFailData), s, true);
            fails.fetch(s);
            if (fails.h[kFailData] != LLONG_MAX) {
                const long long i = fails.h[kFailData];
                throw Failure(AIDW_ERR_DOMAIN, locate_msg(xs[i], ys[i]), i);
            }
            d2h(sorted_ids, h->g.sorted_ids.get(), m, s);
            d2h(cell_start, h->g.cell_start.get(), h->g.cells + 1, s);
            d2h(sorted_x, h->g.sorted_x.get(), m, s);
            d2h(sorted_y, h->g.sorted_y.get(), m, s);
            CK(cudaStreamSynchronize(s));
        }
        // the kNN kernel reads only cell_start, sorted_ids and the interleaved
        // coordinates: the split copies go back to the pool
        h->g.sorted_x.release();
        h->g.sorted_y.release();
        CK(cudaStreamSynchronize(s));
        if (mirror) *mirror = h.release();
    });
}

void aidw_index_release(aidw_index* mirror) { delete mirror; }

int aidw_index_info(const aidw_index* mirror, aidw_grid_config* cfg, size_t* m) {
    if (!mirror) return AIDW_ERR_INVALID_ARGUMENT;
    if (cfg) *cfg = mirror->cfg;
    if (m) *m = mirror->m;
    return AIDW_OK;
}

int aidw_knn_stage_mirror(const double* qx, const double* qy, size_t n, const aidw_index* mirror,
                          int32_t k, double* d2_out, uint32_t* idx_out, double* avg_out,
                          int32_t* k_eff_out, int32_t* exhausted_out, aidw_error* err) {
    return guarded(err, [&] {
        if (!mirror) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "knn_stage: grid engine requires a grid index");
        const size_t m = mirror->m;
        const int k_eff = knn_stage_prologue(n, m, k, true, k_eff_out, exhausted_out);
        if (n == 0) return;
        DeviceScope on(mirror->dev);
        StreamScope ss;
        knn_grid_stage(qx, qy, n, mirror->cfg, mirror->g.cell_start.get(), mirror->g.sorted_ids.get(),
                       mirror->g.sorted_xy.get(), m, k, k_eff, d2_out, idx_out, avg_out, ss.s);
        ss.sync();
    });
}

void* aidw_pinned_alloc(size_t bytes) { return pinned_alloc(bytes); }
void aidw_pinned_free(void* p) { pinned_free(p); }

int aidw_aidw_predict_all(const double* qx, const double* qy, size_t n, const double* dx,
                          const double* dy, const double* dz, size_t m, const double* r_obs,
                          const int64_t* list_len, const uint8_t* exhausted,
                          const aidw_params* params, int32_t variant, int32_t pinned_order,
                          double* pred_out, double* alpha_out, aidw_error* err) {
    return guarded(err, [&] {
        if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set is empty");
        if (!dz) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set carries no values");
        if (!params) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "aidw_predict_all: params missing");
        validate_params(*params);
        if (n == 0) return;
        StreamScope ss;
        cudaStream_t s = ss.s;
        FailFlags fails(s);
        DBuf<double> ddx, ddy, ddz, dqx, dqy, drobs, alpha_q(n, s), pred(n, s), alpha_o(n, s);
        h2d(ddx, dx, m, s);
        h2d(ddy, dy, m, s);
        h2d(ddz, dz, m, s);
        h2d(dqx, qx, n, s);
        h2d(dqy, qy, n, s);
        h2d(drobs, r_obs, n, s);
        DBuf<double> hull(6, s);
        const Extents ext =
            extents(hull.get(), ddx.get(), ddy.get(), m, dqx.get(), dqy.get(), n, ddz.get(), m, s);
        const double area = params->area > 0.0 ? params->area : ext.box.area();
        // adaptive_alpha's host-checkable preconditions, first failing query
        // (adaptive.hpp:101-112): size, area, r_exp, r_obs sign.
        const bool area_ok = area > 0.0 && std::isfinite(area);
        const double r_exp = area_ok ? 1.0 / (2.0 * std::sqrt(static_cast<double>(m) / area)) : 0.0;
        long long host_fail = -1;
        std::string host_msg;
        for (size_t i = 0; i < n && host_fail < 0; ++i) {
            const bool exh = exhausted && exhausted[i];
            if (!exh && list_len && list_len[i] != params->k) {
                host_fail = static_cast<long long>(i);
                host_msg = "adaptive_alpha: kNN result holds " + std::to_string(list_len[i]) +
                           " distances, expected " + std::to_string(params->k);
            } else if (!area_ok) {
                host_fail = static_cast<long long>(i);
                host_msg = "expected_nn_distance: area must be positive finite";
            } else if (!(r_exp > 0.0)) {
                host_fail = static_cast<long long>(i);
                host_msg = "nn_statistic: rExp must be positive";
            } else if (r_obs[i] < 0.0) {
                host_fail = static_cast<long long>(i);
                host_msg = "nn_statistic: rObs must be non-negative";
            }
        }
        const AlphaParams ap = alpha_params_h(*params, r_exp > 0.0 ? r_exp : 1.0);
        run_alpha(drobs.get(), n, ap, alpha_q.get(), fails.slot(kFailAlpha), s);
        fails.fetch(s);
        const long long dev_fail = fails.h[kFailAlpha] == LLONG_MAX ? -1 : fails.h[kFailAlpha];
        if (host_fail >= 0 || dev_fail >= 0) {
            long long i = host_fail;
            std::string msg = host_msg;
            if (i < 0 || (dev_fail >= 0 && dev_fail < i)) {
                i = dev_fail;
                const double R = r_obs[i] / r_exp;
                double mu = R <= params->r_min ? 0.0
                            : R >= params->r_max
                                ? 1.0
                                : 0.5 - 0.5 * std::cos((std::numbers::pi / params->r_max) * (R - params->r_min));
                msg = "alpha_from_mu: mu = " + std::to_string(mu) + " outside [0, 1]";
            }
            throw Failure(AIDW_ERR_RUNTIME, "aidw_predict_all: query " + std::to_string(i) + ": " + msg, i);
        }
        weighting_stage(ddx.get(), ddy.get(), ddz.get(), m, dqx.get(), dqy.get(), n,
                        alpha_q.get(), ext, weight_mode(variant, pinned_order), pred.get(),
                        alpha_o.get(), fails, nullptr, s);
        d2h(pred_out, pred.get(), n, s);
        d2h(alpha_out, alpha_o.get(), n, s);
        ss.sync();
    });
}

int aidw_idw_predict_all(const double* qx, const double* qy, size_t n, const double* dx,
                         const double* dy, const double* dz, size_t m, double alpha,
                         int32_t variant, int32_t pinned_order, double* pred_out,
                         double* alpha_out, aidw_error* err) {
    return guarded(err, [&] {
        if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set is empty");
        if (!dz) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "interpolation: data set carries no values");
        if (!(alpha > 0.0) || !std::isfinite(alpha))
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "idw_predict_all: alpha must be positive finite");
        if (n == 0) return;
        StreamScope ss;
        cudaStream_t s = ss.s;
        FailFlags fails(s);
        DBuf<double> ddx, ddy, ddz, dqx, dqy, alpha_q(n, s), pred(n, s), alpha_o(n, s);
        h2d(ddx, dx, m, s);
        h2d(ddy, dy, m, s);
        h2d(ddz, dz, m, s);
        h2d(dqx, qx, n, s);
        h2d(dqy, qy, n, s);
        DBuf<double> hull(6, s);
        const Extents ext =
            extents(hull.get(), ddx.get(), ddy.get(), m, dqx.get(), dqy.get(), n, ddz.get(), m, s);
        LAUNCH(fill_f64_kernel, ceil_div(n, kThreads), kThreads, 0, s, alpha_q.get(), n, alpha);
        weighting_stage(ddx.get(), ddy.get(), ddz.get(), m, dqx.get(), dqy.get(), n,
                        alpha_q.get(), ext, weight_mode(variant, pinned_order), pred.get(),
                        alpha_o.get(), fails, nullptr, s);
        d2h(pred_out, pred.get(), n, s);
        d2h(alpha_out, alpha_o.get(), n, s);
        ss.sync();
    });
}

int aidw_set_devices(const int32_t* ids, int32_t count, aidw_error* err) {
    return guarded(err, [&] {
        int have = 0;
        CK(cudaGetDeviceCount(&have));
        std::vector<int> v;
        for (int32_t i = 0; i < count; ++i) {
            if (!ids || ids[i] < 0 || ids[i] >= have)
                throw Failure(AIDW_ERR_INVALID_ARGUMENT, "set_devices: no such device");
            v.push_back(ids[i]);
        }
        std::lock_guard<std::mutex> lk(g_dev_mu);
        g_dev_env_read = true;
        g_devices = v;
    });
}

int32_t aidw_device_count(void) {
    const auto d = device_list();
    return static_cast<int32_t>(d.size() > 1 ? d.size() : 1);
}

void aidw_graph_counters(int64_t* captures, int64_t* replays) {
    if (captures) *captures = g_graph_captures.load();
    if (replays) *replays = g_graph_replays.load();
}
void aidw_set_graphs(int32_t enabled) { g_graphs_enabled.store(enabled != 0 ? 1 : 0); }

int64_t aidw_nccl_broadcast_count(void) { return nccl_broadcast_count(); }
int32_t aidw_last_replication(void) { return last_replication_kind(); }
int32_t aidw_nccl_version(void) { return nccl_version(); }

int aidw_run_pipeline(const double* dx, const double* dy, const double* dz, size_t m,
                      const double* qx, const double* qy, size_t n, const aidw_run_config* cfg,
                      double* pred_out, double* alpha_out, aidw_run_stats* stats,
                      aidw_error* err) {
    return guarded(err, [&] {
        if (!cfg) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "run_pipeline: config missing");
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<int> devs = device_list();
        if (devs.size() > 1 && n >= devs.size() && m > 0 && dz) {
            if (pipeline_multi(devs, dx, dy, dz, m, qx, qy, n, *cfg, pred_out, alpha_out, stats, t0))
                return;
            CK(cudaSetDevice(devs[0]));  // a shard failed: one-device run raises the exact error
        }
        StreamScope ss;
        cudaStream_t s = ss.s;
        ArenaScope arena(s);  // uploads in the call's workspace too (graph-replayable)
        DBuf<double> ddx, ddy, ddz, dqx, dqy, pred(n, s), alpha(n, s);
        // the uploads are timed by events on the stream (no synchronisation
        // between them and the pass)
        cudaEvent_t h2d_b, h2d_e;
        h2d_events(h2d_b, h2d_e);
        CK(cudaEventRecord(h2d_b, s));
        h2d(ddx, dx, m, s);
        h2d(ddy, dy, m, s);
        if (dz) h2d(ddz, dz, m, s);
        h2d(dqx, qx, n, s);
        h2d(dqy, qy, n, s);
        CK(cudaEventRecord(h2d_e, s));
        PipelineIO io{ddx.get(), ddy.get(), dz ? ddz.get() : nullptr, dqx.get(), dqy.get(), m, n,
                      pred.get(), alpha.get()};
        pipeline_entry(io, *cfg, stats, s, 0.0, t0, pred_out, alpha_out);
        if (stats) stats->h2d_ms = Events::ms(h2d_b, h2d_e);  // complete: the call synchronised
    });
}

int aidw_run_pipeline_device(const double* d_dx, const double* d_dy, const double* d_dz,
                             size_t m, const double* d_qx, const double* d_qy, size_t n,
                             const aidw_run_config* cfg, double* d_pred, double* d_alpha,
                             aidw_run_stats* stats, void* stream, aidw_error* err) {
    return guarded(err, [&] {
        if (!cfg) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "run_pipeline: config missing");
        const auto t0 = std::chrono::steady_clock::now();
        StreamScope ss(stream);
        PipelineIO io{d_dx, d_dy, d_dz, d_qx, d_qy, m, n, d_pred, d_alpha};
        pipeline_entry(io, *cfg, stats, ss.s, 0.0, t0, nullptr, nullptr);
    });
}

int aidw_raster_lattice_device(size_t nx, size_t ny, const double* bbox, size_t row0,
                               size_t rows, double* d_xs, double* d_ys, void* stream,
                               aidw_error* err) {
    return guarded(err, [&] {
        StreamScope ss(stream);
        lattice_device(nx, ny, bbox, row0, rows, d_xs, d_ys, ss.s);
        ss.sync();
    });
}

int aidw_run_raster(const double* dx, const double* dy, const double* dz, size_t m, size_t nx,
                    size_t ny, const aidw_run_config* cfg, double* raster_out, double* alpha_out,
                    double* bbox_out, aidw_run_stats* stats, aidw_error* err) {
    return guarded(err, [&] {
        if (!cfg) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "run_pipeline: config missing");
        if (nx < 1 || ny < 1)
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "cmd_raster: nx and ny must be >= 1");
        if (m == 0) throw Failure(AIDW_ERR_INVALID_ARGUMENT, "cmd_raster: data set is empty");
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<int> devs = device_list();
        if (devs.size() > 1 && ny >= devs.size() && dz) {
            if (raster_multi(devs, dx, dy, dz, m, nx, ny, *cfg, raster_out, alpha_out, bbox_out,
                             stats, t0))
                return;
            CK(cudaSetDevice(devs[0]));  // a shard failed: one-device run raises the exact error
        }
        StreamScope ss;
        cudaStream_t s = ss.s;
        ArenaScope arena(s);  // uploads and lattice in the call's workspace too
        const size_t n = nx * ny;
        DBuf<double> ddx, ddy, ddz, dqx(n, s), dqy(n, s), pred(n, s), alpha(n, s);
        h2d(ddx, dx, m, s);
        h2d(ddy, dy, m, s);
        if (dz) h2d(ddz, dz, m, s);
        ss.sync();
        const double h2d_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        // the lattice spans bbox(data) (cli.hpp:495); its cell centres lie
        // inside it, so bbox(data ∪ lattice) is the same box
        const Box eb = extents_box(ddx.get(), ddy.get(), m, nullptr, nullptr, 0, s);
        const double bb[4] = {eb.min_x, eb.min_y, eb.max_x, eb.max_y};
        if (bbox_out) std::memcpy(bbox_out, bb, sizeof bb);
        lattice_device(nx, ny, bb, 0, ny, dqx.get(), dqy.get(), s);
        aidw_run_config c = *cfg;
        c.use_bbox = 1;
        std::memcpy(c.bbox, bb, sizeof bb);
        PipelineIO io{ddx.get(), ddy.get(), dz ? ddz.get() : nullptr, dqx.get(), dqy.get(), m, n,
                      pred.get(), alpha.get()};
        pipeline_entry(io, c, stats, s, h2d_ms, t0, raster_out, alpha_out);
    });
}

int aidw_compute_bbox_device(const double* d_dx, const double* d_dy, size_t m,
                             const double* d_qx, const double* d_qy, size_t n, double* out,
                             void* stream, aidw_error* err) {
    return guarded(err, [&] {
        if (m == 0 && n == 0)
            throw Failure(AIDW_ERR_INVALID_ARGUMENT, "compute_bbox: both point sets are empty");
        StreamScope ss(stream);
        const Box e = extents_box(d_dx, d_dy, m, d_qx, d_qy, n, ss.s);
        out[0] = e.min_x;
        out[1] = e.min_y;
        out[2] = e.max_x;
        out[3] = e.max_y;
    });
}

}  // extern "C"
