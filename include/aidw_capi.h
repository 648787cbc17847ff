/*
 * aidw_capi.h — the C-ABI drop-in boundary of the B200 AIDW library
 * (libaidw_b200.so, built from paper_1601_05904_b200/csrc/).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this line.
 * Every batch entry point replaces one function of the reference header
 * library (proj/include/aidw/*.hpp) and is what a binding for that path
 * (ctypes, cgo, JNI, or the C++ shim in include/aidw/*.hpp) calls.
 *
 * Conventions
 *  - Host entry points take HOST pointers and copy to/from HBM inside the
 *    call.  Entry points with the _device suffix take DEVICE pointers that
 *    are already resident on the current CUDA device.
 *  - Return value: AIDW_OK (0) or an aidw_status code.  When `err` is not
 *    NULL it is filled with {code, index, message}; `index` is the smallest
 *    failing query / point (the reference's first-failure rule,
 *    executor.hpp:37-44), or -1.  Codes map 1:1 onto the reference's
 *    exception types (std::invalid_argument, std::domain_error,
 *    std::out_of_range, std::runtime_error); CUDA failures are AIDW_ERR_CUDA.
 *  - All functions are reentrant; each call uses its own stream unless one
 *    is passed.  Results never depend on threading or GPU count.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with AIDW_ERR_CUDA.
 */
#ifndef AIDW_CAPI_H
#define AIDW_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIDW_CAPI_VERSION 1

typedef enum {
    AIDW_OK = 0,
    AIDW_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    AIDW_ERR_DOMAIN = 2,           /* std::domain_error     */
    AIDW_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range     */
    AIDW_ERR_RUNTIME = 4,          /* std::runtime_error (per-query wrap) */
    AIDW_ERR_CUDA = 5              /* device / driver failure             */
} aidw_status;

typedef struct {
    int32_t code;
    int64_t index;
    char message[512];
} aidw_error;

/* GridConfig, proj/include/aidw/grid.hpp:24-34 */
typedef struct {
    double cell_width;
    int32_t n_col;
    int32_t n_row;
    double min_x;
    double min_y;
} aidw_grid_config;

/* AidwParams, proj/include/aidw/types.hpp:91-115 */
typedef struct {
    int32_t k;
    double r_min;
    double r_max;
    double alpha_levels[5];
    double area; /* <= 0: bbox(data ∪ queries) area */
} aidw_params;

enum { AIDW_ENGINE_GRID = 0, AIDW_ENGINE_BRUTE = 1 };     /* KnnEngine, knn.hpp:45          */
enum { AIDW_VARIANT_NAIVE = 0, AIDW_VARIANT_BLOCKED = 1 }; /* Variant, interpolate.hpp:50   */
enum { AIDW_MODE_IDW = 0, AIDW_MODE_AIDW = 1 };           /* cli::Mode, cli.hpp:26          */

/* Weighting precision of Variant::blocked.  FP32 (default) is the MUFU
 * kernel with the 1e-5 contract; FP64 routes blocked to the FP64 kernel
 * (chunk-ordered FP64 partial sums: index order within each data chunk,
 * chunks added in order; pow, or 1 / (d2 d2) at alpha == 4), as
 * Variant::naive and pinned_order always are.  The
 * environment variable AIDW_WEIGHT_FP64=1 sets FP64 at library load. */
enum { AIDW_PRECISION_FP32 = 0, AIDW_PRECISION_FP64 = 1 };

/* RunConfig, proj/include/aidw/cli.hpp:30-43 (file paths and seed omitted:
 * they belong to the CLI, not to the pipeline). */
typedef struct {
    int32_t mode;      /* AIDW_MODE_*    */
    int32_t engine;    /* AIDW_ENGINE_*  */
    int32_t variant;   /* AIDW_VARIANT_* */
    aidw_params params;
    double alpha;       /* constant exponent, idw mode */
    double cell_factor; /* cell width = factor * expected NN distance */
    int32_t workers;    /* accepted and ignored (CPU threading knob) */
    /* B200 additions (zero-initialise for reference behaviour): */
    int32_t use_bbox;   /* 1: take bbox[] as bbox(data ∪ queries) — used by
                           query-sharded multi-GPU runs so every rank sees
                           the global box (identical grid, area, snap) */
    double bbox[4];     /* min_x, min_y, max_x, max_y */
} aidw_run_config;

/* StageTimings, proj/include/aidw/executor.hpp:137-150, plus device detail. */
typedef struct {
    double build_ms;   /* grid build (K1), CUDA events              */
    double knn_ms;     /* query sort + kNN + alpha (K2+K3)          */
    double interp_ms;  /* weighting stage (K4 + settle)             */
    double total_ms;   /* whole call incl. host<->device copies      */
    double weight_kernel_ms; /* K4 launches only (roofline numerator) */
    double knn_kernel_ms;    /* K2 launch only                        */
    double h2d_ms, d2h_ms;
    int32_t k_effective;
    int32_t worker_count;
    int64_t pairs;           /* m * n weighting pairs evaluated        */
    int64_t knn_candidates;  /* candidates scanned by K2 (sum over queries) */
    int64_t knn_ref_candidates; /* candidates the reference scans: final-level blocks */
    int64_t alpha4_queries;  /* queries on the exact alpha = 4 recipe  */
    int64_t kernel_launches; /* kernels launched by this call          */
} aidw_run_stats;

/* ------------------------------------------------------------ info */
int aidw_capi_version(void);
/* Number of kernels this library has launched since load (all threads). */
int64_t aidw_kernel_launch_count(void);
/* Device name / SM count of the current device; fails without CUDA. */
int aidw_device_info(char* name, size_t cap, int32_t* sm_count, aidw_error* err);
void aidw_set_weight_precision(int32_t precision);
int32_t aidw_get_weight_precision(void);
/* 1 (default): queries with alpha == 4 exactly take the one-MUFU recipe
 * w = 1/(d2*d2) (the reference's half-integer recipe, interpolate.hpp:
 * 174-209); 0: every query takes the general exp2/log2 path (used to report
 * the general-alpha roofline separately). */
void aidw_set_alpha4_recipe(int32_t enabled);

/* Queries per weighting launch (K4 + settle).  The weighting keeps FP64
 * partial sums of 16 B x data chunks per query in flight; the query set is
 * processed in slabs so that memory is bounded by the slab, not by n
 * (default 0: 2 GiB of partials, 4M queries at 32 chunks).  Rounded down to
 * a multiple of 1024, at least 1024.  Results never depend on it. */
void aidw_set_query_slab(int64_t queries);

/* Weighting engine of the FP32 path for m data points (a function of m
 * alone, so results never depend on n, the shard or the GPU count):
 * 1 — recipe-class queries on the tensor-core engine (far-form d2 by tcgen05
 * MMA, weight_tc.cu) and general-alpha queries on the CUDA-core K4 beside it;
 * 0 — every query on the CUDA-core K4 (weight.cu; small m). */
int32_t aidw_weight_engine(int64_t m);

/* ------------------------------------------------------------ grid (K1) */
/* build_index — grid.hpp:176-213.  sorted_ids/sorted_x/sorted_y: m entries,
 * cell_start: n_col*n_row + 1 entries (exclusive prefix). */
int aidw_build_index(const double* xs, const double* ys, size_t m, const aidw_grid_config* cfg,
                     uint32_t* sorted_ids, uint32_t* cell_start, double* sorted_x,
                     double* sorted_y, aidw_error* err);

/* Device mirror of a GridIndex ("an extra opaque device-mirror
 * handle member in GridIndex lets the GPU cache uploads").  Same outputs as
 * aidw_build_index; in addition *mirror receives a handle that keeps the
 * index's CSR arrays resident in HBM (cell_start, sorted_ids, interleaved
 * sorted coordinates) on the calling thread's device, so knn_stage calls on
 * this index upload only their queries.  Release with aidw_index_release
 * (NULL is a no-op).  The handle is immutable and may be shared by threads. */
typedef struct aidw_index aidw_index;
int aidw_build_index_mirror(const double* xs, const double* ys, size_t m,
                            const aidw_grid_config* cfg, uint32_t* sorted_ids,
                            uint32_t* cell_start, double* sorted_x, double* sorted_y,
                            aidw_index** mirror, aidw_error* err);
void aidw_index_release(aidw_index* mirror);
/* the mirror's grid (cfg) and point count, for validation by the caller */
int aidw_index_info(const aidw_index* mirror, aidw_grid_config* cfg, size_t* m);

/* Page-locked host staging from a process-wide cache (cudaHostAlloc'ed
 * blocks are recycled: pinning is slow, copies from / to pinned memory run
 * at full PCIe / C2C speed).  NULL if no device / allocation failed (the
 * caller then uses pageable memory).  Free with aidw_pinned_free. */
void* aidw_pinned_alloc(size_t bytes);
void aidw_pinned_free(void* p);

/* ------------------------------------------------------------ kNN (K2) */
/* knn_stage — knn.hpp:255-271.  Grid engine: pass the GridIndex arrays from
 * build_index (cfg, cell_start, sorted_ids, sorted_x, sorted_y); brute
 * engine: they may be NULL.  Outputs (k_eff = min(k, m) for the grid
 * engine; brute requires k <= m):
 *   d2_out   n * k_eff squared distances, ascending (KnnResult::distances_sq)
 *   idx_out  n * k_eff data indices, (d2, idx)-lexicographic (nullable)
 *   avg_out  n  KnnResult::average_distance
 *   *k_eff_out, *exhausted_out (KnnResult::exhausted, same for all queries) */
int aidw_knn_stage(const double* qx, const double* qy, size_t n, const aidw_grid_config* cfg,
                   const uint32_t* cell_start, const uint32_t* sorted_ids,
                   const double* sorted_x, const double* sorted_y, const double* dx,
                   const double* dy, size_t m, int32_t k, int32_t engine, double* d2_out,
                   uint32_t* idx_out, double* avg_out, int32_t* k_eff_out,
                   int32_t* exhausted_out, aidw_error* err);

/* knn_stage, grid engine, on a device-mirrored index (aidw_build_index_mirror):
 * identical outputs to aidw_knn_stage with that index's arrays. */
int aidw_knn_stage_mirror(const double* qx, const double* qy, size_t n, const aidw_index* mirror,
                          int32_t k, double* d2_out, uint32_t* idx_out, double* avg_out,
                          int32_t* k_eff_out, int32_t* exhausted_out, aidw_error* err);

/* ------------------------------------------------------------ weighting (K3+K4) */
/* aidw_predict_all — interpolate.hpp:453-489.  Per query i the caller's
 * KnnResult is summarised as r_obs[i] (average_distance), list_len[i]
 * (size()) and exhausted[i]. */
int aidw_aidw_predict_all(const double* qx, const double* qy, size_t n, const double* dx,
                          const double* dy, const double* dz, size_t m, const double* r_obs,
                          const int64_t* list_len, const uint8_t* exhausted,
                          const aidw_params* params, int32_t variant, int32_t pinned_order,
                          double* pred_out, double* alpha_out, aidw_error* err);

/* idw_predict_all — interpolate.hpp:426-448 (constant alpha). */
int aidw_idw_predict_all(const double* qx, const double* qy, size_t n, const double* dx,
                         const double* dy, const double* dz, size_t m, double alpha,
                         int32_t variant, int32_t pinned_order, double* pred_out,
                         double* alpha_out, aidw_error* err);

/* ------------------------------------------------------------ devices */
/* Devices aidw_run_pipeline / aidw_run_raster spread over (SURVEY §8e:
 * one process, one host thread per device, query or lattice-row shards,
 * data replicated, the global bbox combined before any grid is built ->
 * results bit-identical to one device).  Default: the current device only,
 * or AIDW_DEVICES="0,1,..." from the environment; a list may repeat a
 * device.  count <= 1 restores the single-device default. */
int aidw_set_devices(const int32_t* ids, int32_t count, aidw_error* err);
/* Number of devices the pipeline calls use (>= 1). */
int32_t aidw_device_count(void);

/* Multi-device data replication: the data arrays go host ->
 * first listed device once, then ncclBroadcast (ncclCommInitAll over the
 * distinct devices, cached) to the others; shards on one device share its
 * replica.  NCCL is dlopen'ed ("libnccl.so.2"); without it CUDA peer copies
 * fill the replicas.  Introspection for tests and logs: */
/* CUDA-graph cache of fused passes (a pass with the plan, buffers and
 * workspace of an earlier one is replayed as one graph launch; AIDW_GRAPHS=0
 * or aidw_set_graphs(0) disables it): captures and replays so far. */
void aidw_graph_counters(int64_t* captures, int64_t* replays);
void aidw_set_graphs(int32_t enabled);

int64_t aidw_nccl_broadcast_count(void); /* grouped broadcasts issued so far   */
int32_t aidw_last_replication(void);     /* 0 none, 1 NCCL broadcast, 2 peer   */
int32_t aidw_nccl_version(void);         /* NCCL_VERSION_CODE, 0 if unloadable */

/* ------------------------------------------------------------ pipeline */
/* cli::run_pipeline — cli.hpp:217-268, fused and device-resident between
 * stages (no per-query KnnResult materialisation).  Host buffers. */
int aidw_run_pipeline(const double* dx, const double* dy, const double* dz, size_t m,
                      const double* qx, const double* qy, size_t n, const aidw_run_config* cfg,
                      double* pred_out, double* alpha_out, aidw_run_stats* stats,
                      aidw_error* err);

/* Same pipeline over DEVICE-resident inputs/outputs (current device).
 * `stream` is a cudaStream_t (NULL = the library's own stream, ordered after
 * the work already queued on the legacy default stream). */
int aidw_run_pipeline_device(const double* d_dx, const double* d_dy, const double* d_dz,
                             size_t m, const double* d_qx, const double* d_qy, size_t n,
                             const aidw_run_config* cfg, double* d_pred, double* d_alpha,
                             aidw_run_stats* stats, void* stream, aidw_error* err);

/* bbox(data ∪ queries) of device-resident sets (types.hpp:124-143);
 * out = {min_x, min_y, max_x, max_y}.  For sharded runs: all-reduce MIN/MAX
 * of the per-rank boxes, then pass the result as aidw_run_config.bbox. */
int aidw_compute_bbox_device(const double* d_dx, const double* d_dy, size_t m,
                             const double* d_qx, const double* d_qy, size_t n, double* out,
                             void* stream, aidw_error* err);

/* ------------------------------------------------------------ raster (cmd_raster) */
/* cmd_raster's lattice (cli.hpp:496-507) generated on the device: rows
 * [row0, row0 + rows) of the nx x ny lattice over bbox = {min_x, min_y,
 * max_x, max_y}, row-major, northernmost row first (row 0).  Device
 * buffers of nx * rows doubles; `stream` as aidw_run_pipeline_device. */
int aidw_raster_lattice_device(size_t nx, size_t ny, const double* bbox, size_t row0,
                               size_t rows, double* d_xs, double* d_ys, void* stream,
                               aidw_error* err);

/* The compute part of cli::cmd_raster (cli.hpp:484-524) without file I/O:
 * data (host buffers) -> lattice over bbox(data) generated in HBM ->
 * the fused run_pipeline -> raster_out[nx * ny] (north-first, row-major;
 * = Raster::values).  alpha_out may be NULL; bbox_out (4 doubles, may be
 * NULL) receives the lattice box (Raster::xllcorner = bbox_out[0],
 * yllcorner = bbox_out[1], cellsize = (max_x - min_x) / nx). */
int aidw_run_raster(const double* dx, const double* dy, const double* dz, size_t m, size_t nx,
                    size_t ny, const aidw_run_config* cfg, double* raster_out, double* alpha_out,
                    double* bbox_out, aidw_run_stats* stats, aidw_error* err);

/* ------------------------------------------------------------ files (io.hpp) */
/* The file formats either side of the path, same bytes and diagnostics as
 * proj/include/aidw/io.hpp, parsed / formatted on all host threads.
 * Parse and I/O failures -> AIDW_ERR_RUNTIME with the reference's
 * "<path>:<line>: ..." message; non-finite values -> AIDW_ERR_INVALID_ARGUMENT
 * (validate_finite, types.hpp:146-159). */
typedef struct aidw_points_buffer {
    double* xs;
    double* ys;
    double* zs; /* NULL for query files */
    size_t count;
} aidw_points_buffer;

/* read_data_csv (with_values = 1, header "x,y,z") / read_query_csv
 * (with_values = 0, header "x,y") — io.hpp:103-145.  The library allocates
 * the arrays; release them with aidw_free_points. */
int aidw_read_points_csv(const char* path, int32_t with_values, aidw_points_buffer* out,
                         aidw_error* err);
void aidw_free_points(aidw_points_buffer* buf);

/* write_data_csv / write_query_csv / write_result_csv (io.hpp:146-188):
 * `header` then `rows` lines of ncols "%.17g" fields; cols[c][r]. */
int aidw_write_columns_csv(const char* path, const char* header, size_t rows, int32_t ncols,
                           const double* const* cols, aidw_error* err);

/* write_raster_asc (io.hpp:199-221): the ESRI ASCII grid, byte-identical to
 * the reference writer ("%.17g" values). */
int aidw_write_raster_asc(const char* path, size_t ncols, size_t nrows, double xllcorner,
                          double yllcorner, double cellsize, const double* values,
                          aidw_error* err);

typedef struct aidw_raster_buffer {
    size_t ncols, nrows;
    double xllcorner, yllcorner, cellsize;
    double* values; /* nrows * ncols, north-first; free with aidw_free_raster */
    size_t count;
} aidw_raster_buffer;

/* parse_raster_asc (io.hpp:223-253). */
int aidw_read_raster_asc(const char* path, aidw_raster_buffer* out, aidw_error* err);
void aidw_free_raster(aidw_raster_buffer* buf);

/* ------------------------------------------------------------ synthetic inputs */
/* generate_random_points / generate_random_queries — generate.hpp:45-95
 * (mt19937_64, 53-bit unit doubles; rule 0 uniform, 1 planar, 2 radial). */
int aidw_generate_points(size_t count, const double* bbox, uint64_t seed, int32_t rule,
                         double* xs, double* ys, double* zs, aidw_error* err);
int aidw_generate_queries(size_t count, const double* bbox, uint64_t seed, double* xs,
                          double* ys, aidw_error* err);
/* Clustered (Gaussian-blob) points for BASELINE config 4 (the
 * reference has no such generator).  zs may be NULL for query sets. */
int aidw_generate_clustered(size_t count, int32_t blobs, double sigma, uint64_t center_seed,
                            uint64_t seed, double* xs, double* ys, double* zs, aidw_error* err);
/* cmd_raster lattice (cli.hpp:496-507): nx*ny cell centres over bbox,
 * northernmost row first, row-major. */
int aidw_raster_lattice(size_t nx, size_t ny, const double* bbox, double* xs, double* ys,
                        aidw_error* err);

#ifdef __cplusplus
}
#endif

#endif /* AIDW_CAPI_H */
