"""Python mirror of the reference's public API for the AIDW path.

Same names, argument meaning and error behaviour as proj/include/aidw/*.hpp
(build_index, knn_stage, aidw_predict_all, idw_predict_all,
cli::run_pipeline, the generators), implemented over the C-ABI
(include/aidw_capi.h) so tests read like the reference's own tests.
Exceptions mirror the C++ types:

    std::invalid_argument -> InvalidArgument (ValueError)
    std::domain_error     -> DomainError     (ValueError)
    std::out_of_range     -> OutOfRange      (IndexError)
    std::runtime_error    -> AidwRuntimeError (RuntimeError)
    CUDA failure          -> CudaError       (RuntimeError)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class InvalidArgument(ValueError):
    pass


class DomainError(ValueError):
    pass


class OutOfRange(IndexError):
    pass


class AidwRuntimeError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {L.AIDW_ERR_INVALID_ARGUMENT: InvalidArgument, L.AIDW_ERR_DOMAIN: DomainError,
        L.AIDW_ERR_OUT_OF_RANGE: OutOfRange, L.AIDW_ERR_RUNTIME: AidwRuntimeError,
        L.AIDW_ERR_CUDA: CudaError}


def _raise(rc, err):
    if rc != L.AIDW_OK:
        exc = _EXC.get(rc, AidwRuntimeError)(err.message.decode(errors="replace"))
        exc.index = int(err.index)
        raise exc


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=L._dp):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------ types
@dataclass
class PointSet:
    """SoA point container (types.hpp:34-66); zs empty for query sets."""
    xs: np.ndarray = field(default_factory=lambda: np.empty(0))
    ys: np.ndarray = field(default_factory=lambda: np.empty(0))
    zs: np.ndarray = field(default_factory=lambda: np.empty(0))

    def __post_init__(self):
        self.xs, self.ys, self.zs = _f64(self.xs), _f64(self.ys), _f64(self.zs)

    def count(self):
        return int(self.xs.size)

    def has_values(self):
        return self.zs.size > 0


@dataclass
class BoundingBox:
    min_x: float = 0.0
    min_y: float = 0.0
    max_x: float = 0.0
    max_y: float = 0.0

    def as_array(self):
        return np.array([self.min_x, self.min_y, self.max_x, self.max_y], np.float64)


@dataclass
class AidwParams:
    """types.hpp:91-115."""
    k: int = 15
    r_min: float = 0.0
    r_max: float = 2.0
    alpha_levels: tuple = (0.5, 1.0, 2.0, 3.0, 4.0)
    area: float = 0.0

    def c(self):
        p = L.Params()
        p.k, p.r_min, p.r_max, p.area = int(self.k), self.r_min, self.r_max, self.area
        for i, v in enumerate(self.alpha_levels):
            p.alpha_levels[i] = v
        return p


GridConfig = L.GridConfig


class _Mirror:
    """Owner of an aidw_index device mirror (released when collected)."""
    def __init__(self, handle, print_):
        self.handle, self.print = handle, print_

    def __del__(self):
        if self.handle:
            lib().aidw_index_release(self.handle)
            self.handle = None


def _fingerprint(cfg, arrays):
    """Sizes, grid and 64 sampled entries per array (cf. GridIndex::fingerprint)."""
    parts = [cfg.cell_width, cfg.n_col, cfg.n_row, cfg.min_x, cfg.min_y]
    for a in arrays:
        step = max(1, a.size // 64)
        parts.append(a.size)
        parts.append(a[::step].tobytes() + (a[-1:].tobytes() if a.size else b""))
    return hash(tuple(parts))


@dataclass
class GridIndex:
    """grid.hpp:131-171 (CSR cell layout), plus the device mirror build_index
    leaves in HBM (knn_stage reuses it while the arrays are unchanged)."""
    config: L.GridConfig
    sorted_point_ids: np.ndarray
    cell_start: np.ndarray
    sorted_x: np.ndarray
    sorted_y: np.ndarray
    device_mirror: _Mirror | None = None

    def mirror(self):
        m = self.device_mirror
        if m is None or m.print != _fingerprint(self.config, self._arrays()):
            return None
        return m.handle

    def _arrays(self):
        return (self.sorted_point_ids, self.cell_start, self.sorted_x, self.sorted_y)

    def point_count(self):
        return int(self.sorted_point_ids.size)

    def cell_count(self, c):
        return int(self.cell_start[c + 1]) - int(self.cell_start[c])


@dataclass
class KnnStageResult:
    """Flat form of std::vector<KnnResult> (knn.hpp:36-42): row i holds query
    i's ascending squared distances; `indices` the (d2, idx)-lexicographic
    neighbour ids; `average_distance`; `exhausted` (same for every query)."""
    distances_sq: np.ndarray
    indices: np.ndarray
    average_distance: np.ndarray
    exhausted: bool
    k_effective: int

    def __len__(self):
        return int(self.average_distance.size)


@dataclass
class InterpolationResult:
    predicted: np.ndarray
    alphas: np.ndarray


@dataclass
class RunConfig:
    """cli.hpp:30-43 (pipeline fields)."""
    mode: str = "aidw"
    knn_engine: str = "grid"
    variant: str = "blocked"
    params: AidwParams = field(default_factory=AidwParams)
    alpha: float = 2.0
    cell_factor: float = 4.0
    workers: int = 1
    bbox: tuple | None = None  # B200 addition: global bbox for sharded runs

    def c(self):
        r = L.RunConfig()
        r.mode = L.MODE_IDW if self.mode == "idw" else L.MODE_AIDW
        r.engine = L.ENGINE_BRUTE if self.knn_engine == "brute" else L.ENGINE_GRID
        r.variant = L.VARIANT_NAIVE if self.variant == "naive" else L.VARIANT_BLOCKED
        r.params = self.params.c()
        r.alpha, r.cell_factor, r.workers = self.alpha, self.cell_factor, int(self.workers)
        if self.bbox is not None:
            r.use_bbox = 1
            for i, v in enumerate(self.bbox):
                r.bbox[i] = v
        return r


@dataclass
class PipelineOutcome:
    result: InterpolationResult
    stats: dict
    k_effective: int


# ------------------------------------------------------------------ helpers
def lib():
    return L.load()


def device_info():
    name = C.create_string_buffer(256)
    sm = C.c_int32()
    err = L.Error()
    _raise(lib().aidw_device_info(name, 256, C.byref(sm), C.byref(err)), err)
    return name.value.decode(), sm.value


def set_weight_precision(p: str):
    lib().aidw_set_weight_precision(L.PRECISION_FP64 if p == "fp64" else L.PRECISION_FP32)


def set_alpha4_recipe(enabled: bool):
    lib().aidw_set_alpha4_recipe(1 if enabled else 0)


def set_query_slab(queries: int = 0):
    """Queries per weighting launch (0 = default: 2 GiB of FP64 partials).
    Bounds the weighting's memory for any n; results never depend on it."""
    lib().aidw_set_query_slab(int(queries))


def weight_engine(m: int) -> str:
    """FP32 weighting engine for m data points: "tensor-core" (recipe
    queries' far-form d2 by tcgen05 MMA) or "cuda-core"."""
    return "tensor-core" if lib().aidw_weight_engine(int(m)) else "cuda-core"


def set_devices(ids) -> None:
    """Devices run_pipeline / run_raster spread over, one host thread each
    (query / lattice-row shards; results bit-identical to one device).
    [] or a single id restores the single-device default."""
    ids = list(ids)
    arr = (C.c_int32 * max(1, len(ids)))(*ids)
    err = L.Error()
    _raise(lib().aidw_set_devices(arr, len(ids), C.byref(err)), err)


def device_count() -> int:
    return int(lib().aidw_device_count())


def graph_counters() -> dict:
    """CUDA-graph cache of fused passes: captures and replays so far."""
    c, r = C.c_int64(), C.c_int64()
    lib().aidw_graph_counters(C.byref(c), C.byref(r))
    return {"captures": int(c.value), "replays": int(r.value)}


def set_graphs(enabled: bool):
    """Enable / disable the CUDA-graph cache (results never depend on it)."""
    lib().aidw_set_graphs(1 if enabled else 0)


def replication_info() -> dict:
    """How the last multi-device run replicated the data: NCCL
    broadcasts issued so far, the last replication kind and NCCL's version."""
    kinds = {0: "none", 1: "nccl_broadcast", 2: "peer_copy"}
    return {"nccl_broadcasts": int(lib().aidw_nccl_broadcast_count()),
            "last": kinds.get(int(lib().aidw_last_replication()), "?"),
            "nccl_version": int(lib().aidw_nccl_version())}


def kernel_launch_count():
    return int(lib().aidw_kernel_launch_count())


# ------------------------------------------------------------------ generators
def generate_random_points(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=42, rule="uniform"):
    rule_id = {"uniform": 0, "planar": 1, "radial": 2}[rule] if isinstance(rule, str) else int(rule)
    xs, ys, zs = np.empty(count), np.empty(count), np.empty(count)
    bb = _f64(bbox)
    err = L.Error()
    _raise(lib().aidw_generate_points(count, _p(bb), seed, rule_id, _p(xs), _p(ys), _p(zs),
                                      C.byref(err)), err)
    return PointSet(xs, ys, zs)


def generate_random_queries(count, bbox=(0.0, 0.0, 1.0, 1.0), seed=43):
    xs, ys = np.empty(count), np.empty(count)
    bb = _f64(bbox)
    err = L.Error()
    _raise(lib().aidw_generate_queries(count, _p(bb), seed, _p(xs), _p(ys), C.byref(err)), err)
    return PointSet(xs, ys)


def generate_clustered(count, blobs=20, sigma=0.03, center_seed=5, seed=42, with_values=True):
    xs, ys = np.empty(count), np.empty(count)
    zs = np.empty(count) if with_values else None
    err = L.Error()
    _raise(lib().aidw_generate_clustered(count, blobs, sigma, center_seed, seed, _p(xs), _p(ys),
                                         _p(zs) if zs is not None else None, C.byref(err)), err)
    return PointSet(xs, ys, zs if zs is not None else np.empty(0))


def raster_lattice(nx, ny, bbox):
    xs, ys = np.empty(nx * ny), np.empty(nx * ny)
    bb = _f64(bbox)
    err = L.Error()
    _raise(lib().aidw_raster_lattice(nx, ny, _p(bb), _p(xs), _p(ys), C.byref(err)), err)
    return PointSet(xs, ys)


# ------------------------------------------------------------------ host set-up helpers
def compute_bbox(data: PointSet, queries: PointSet | None = None) -> BoundingBox:
    """types.hpp:124-143 (host; both sets already in host memory)."""
    xs = np.concatenate([data.xs, queries.xs if queries is not None else np.empty(0)])
    ys = np.concatenate([data.ys, queries.ys if queries is not None else np.empty(0)])
    if xs.size == 0:
        raise InvalidArgument("compute_bbox: both point sets are empty")
    return BoundingBox(float(np.nanmin(xs)), float(np.nanmin(ys)), float(np.nanmax(xs)),
                       float(np.nanmax(ys)))


def choose_cell_width(data: PointSet, bbox: BoundingBox, factor: float) -> float:
    """grid.hpp:50-64."""
    m = data.count()
    w, h = bbox.max_x - bbox.min_x, bbox.max_y - bbox.min_y
    if m == 0:
        raise InvalidArgument("choose_cell_width: data set is empty")
    if not (bbox.min_x <= bbox.max_x and bbox.min_y <= bbox.max_y) or not (w * h > 0.0):
        raise InvalidArgument("choose_cell_width: bbox must have positive area")
    if not (factor > 0.0) or not np.isfinite(factor):
        raise InvalidArgument("choose_cell_width: factor must be positive finite")
    return factor * (1.0 / (2.0 * np.sqrt(m / (w * h))))


def make_grid_config(bbox: BoundingBox, cell_width: float) -> L.GridConfig:
    """grid.hpp:67-88."""
    w, h = bbox.max_x - bbox.min_x, bbox.max_y - bbox.min_y
    if not (bbox.min_x <= bbox.max_x and bbox.min_y <= bbox.max_y) or not (w * h > 0.0):
        raise InvalidArgument("make_grid_config: bbox must have positive area")
    if not (cell_width > 0.0) or not np.isfinite(cell_width):
        raise InvalidArgument("make_grid_config: cellWidth must be positive finite")
    cols = np.floor((bbox.max_x - bbox.min_x + cell_width) / cell_width)
    rows = np.floor((bbox.max_y - bbox.min_y + cell_width) / cell_width)
    if cols * rows > 1.0e9:
        raise InvalidArgument(f"make_grid_config: cellWidth {cell_width} yields more than 1e9 cells")
    return L.GridConfig(cell_width, max(1, int(cols)), max(1, int(rows)), bbox.min_x, bbox.min_y)


# ------------------------------------------------------------------ batch entry points
def build_index(data: PointSet, config: L.GridConfig) -> GridIndex:
    """grid.hpp:176-213 on the GPU (K1)."""
    m = data.count()
    cells = config.cell_total()
    ids = np.empty(m, np.uint32)
    cs = np.empty(cells + 1 if m else 1, np.uint32)
    sx, sy = np.empty(m), np.empty(m)
    err = L.Error()
    handle = C.c_void_p()
    _raise(lib().aidw_build_index_mirror(_p(data.xs), _p(data.ys), m, C.byref(config),
                                         _p(ids, L._u32p), _p(cs, L._u32p), _p(sx), _p(sy),
                                         C.byref(handle), C.byref(err)), err)
    g = GridIndex(config, ids, cs, sx, sy)
    if handle.value:
        g.device_mirror = _Mirror(handle.value, _fingerprint(config, g._arrays()))
    return g


def knn_stage(queries: PointSet, index: GridIndex | None, data: PointSet, k: int,
              engine: str = "grid", workers: int = 1, chunk: int = 64) -> KnnStageResult:
    """knn.hpp:255-271 on the GPU (K2).  `workers` / `chunk` are accepted and
    ignored (CPU threading knobs; results never depend on them)."""
    n = queries.count()
    grid = engine == "grid"
    if grid and index is None:
        raise InvalidArgument("knn_stage: grid engine requires a grid index")
    m = index.point_count() if grid else data.count()
    k_eff = min(k, m) if grid else k
    k_alloc = max(k_eff, 0)
    d2 = np.empty((n, k_alloc))
    idx = np.empty((n, k_alloc), np.uint32)
    avg = np.empty(n)
    ke, ex = C.c_int32(), C.c_int32()
    err = L.Error()
    mirror = index.mirror() if grid else None
    if mirror:  # the index's arrays are resident in HBM: upload only the queries
        _raise(lib().aidw_knn_stage_mirror(_p(queries.xs), _p(queries.ys), n, mirror, int(k),
                                           _p(d2), _p(idx, L._u32p), _p(avg), C.byref(ke),
                                           C.byref(ex), C.byref(err)), err)
        return KnnStageResult(d2, idx, avg, bool(ex.value), int(ke.value))
    if grid:
        cfg = index.config
        args = (C.byref(cfg), _p(index.cell_start, L._u32p), _p(index.sorted_point_ids, L._u32p),
                _p(index.sorted_x), _p(index.sorted_y), None, None)
    else:
        args = (None, None, None, None, None, _p(data.xs), _p(data.ys))
    _raise(lib().aidw_knn_stage(_p(queries.xs), _p(queries.ys), n, *args, m, int(k),
                                L.ENGINE_GRID if grid else L.ENGINE_BRUTE, _p(d2),
                                _p(idx, L._u32p), _p(avg), C.byref(ke), C.byref(ex),
                                C.byref(err)), err)
    return KnnStageResult(d2, idx, avg, bool(ex.value), int(ke.value))


def aidw_predict_all(queries: PointSet, data: PointSet, knn, params: AidwParams,
                     variant: str = "blocked", workers: int = 1,
                     pinned_order: bool = False) -> InterpolationResult:
    """interpolate.hpp:453-489 on the GPU (K3 + K4).  `knn` is a
    KnnStageResult or a sequence of objects with distances_sq /
    average_distance / exhausted (the reference's KnnResult)."""
    n = queries.count()
    if isinstance(knn, KnnStageResult):
        count = len(knn)
        r_obs = _f64(knn.average_distance)
        lens = np.full(count, knn.k_effective, np.int64)
        exh = np.full(count, 1 if knn.exhausted else 0, np.uint8)
    else:
        count = len(knn)
        r_obs = _f64([r.average_distance for r in knn])
        lens = np.array([len(r.distances_sq) for r in knn], np.int64)
        exh = np.array([1 if r.exhausted else 0 for r in knn], np.uint8)
    if data.count() == 0:
        raise InvalidArgument("interpolation: data set is empty")
    if not data.has_values():
        raise InvalidArgument("interpolation: data set carries no values")
    if count != n:
        raise InvalidArgument(f"aidw_predict_all: {count} kNN results for {n} queries")
    pred, alph = np.empty(n), np.empty(n)
    p = params.c()
    err = L.Error()
    _raise(lib().aidw_aidw_predict_all(_p(queries.xs), _p(queries.ys), n, _p(data.xs),
                                       _p(data.ys), _p(data.zs), data.count(), _p(r_obs),
                                       _p(lens, L._i64p), _p(exh, L._u8p), C.byref(p),
                                       L.VARIANT_NAIVE if variant == "naive" else L.VARIANT_BLOCKED,
                                       int(bool(pinned_order)), _p(pred), _p(alph),
                                       C.byref(err)), err)
    return InterpolationResult(pred, alph)


def idw_predict_all(queries: PointSet, data: PointSet, alpha: float, variant: str = "blocked",
                    workers: int = 1, pinned_order: bool = False) -> InterpolationResult:
    """interpolate.hpp:426-448 on the GPU (K4, constant alpha)."""
    n = queries.count()
    pred, alph = np.empty(n), np.empty(n)
    err = L.Error()
    zs = data.zs if data.has_values() else None
    _raise(lib().aidw_idw_predict_all(_p(queries.xs), _p(queries.ys), n, _p(data.xs),
                                      _p(data.ys), _p(zs) if zs is not None else None,
                                      data.count(), float(alpha),
                                      L.VARIANT_NAIVE if variant == "naive" else L.VARIANT_BLOCKED,
                                      int(bool(pinned_order)), _p(pred), _p(alph),
                                      C.byref(err)), err)
    return InterpolationResult(pred, alph)


def run_pipeline(data: PointSet, queries: PointSet, cfg: RunConfig, out=None) -> PipelineOutcome:
    """cli::run_pipeline (cli.hpp:217-268), fused on the GPU; host buffers.
    `out` = optional (pred, alpha) float64 arrays of length n to write into
    (e.g. pinned host memory, as the C-ABI allows)."""
    n = queries.count()
    if out is not None:
        pred, alph = out
        if pred.dtype != np.float64 or alph.dtype != np.float64 or len(pred) != n or \
                len(alph) != n or not pred.flags.c_contiguous or not alph.flags.c_contiguous:
            raise InvalidArgument("run_pipeline: out arrays must be contiguous float64 of length n")
    else:
        pred, alph = np.empty(n), np.empty(n)
    st = L.RunStats()
    c = cfg.c()
    err = L.Error()
    zs = data.zs if data.has_values() else None
    _raise(lib().aidw_run_pipeline(_p(data.xs), _p(data.ys), _p(zs) if zs is not None else None,
                                   data.count(), _p(queries.xs), _p(queries.ys), n, C.byref(c),
                                   _p(pred), _p(alph), C.byref(st), C.byref(err)), err)
    return PipelineOutcome(InterpolationResult(pred, alph), st.as_dict(), int(st.k_effective))


def run_pipeline_device(d_dx, d_dy, d_dz, m, d_qx, d_qy, n, cfg, d_pred, d_alpha,
                        stream=None, raw=False):
    """Device-resident pipeline over raw device pointers (ints); returns stats
    (a dict, or with raw=True the C struct — convert later with .as_dict()).
    `cfg` is a RunConfig or an already converted L.RunConfig (cfg.c())."""
    st = L.RunStats()
    c = cfg.c() if isinstance(cfg, RunConfig) else cfg
    err = L.Error()
    _raise(lib().aidw_run_pipeline_device(d_dx, d_dy, d_dz, m, d_qx, d_qy, n, C.byref(c), d_pred,
                                          d_alpha, C.byref(st), stream, C.byref(err)), err)
    return st if raw else st.as_dict()


@dataclass
class Raster:
    """io.hpp:190-197: ncols x nrows values, northernmost row first."""
    ncols: int
    nrows: int
    xllcorner: float
    yllcorner: float
    cellsize: float
    values: np.ndarray  # (nrows * ncols,), row-major

    def grid(self) -> np.ndarray:
        return self.values.reshape(self.nrows, self.ncols)


@dataclass
class RasterOutcome:
    """cli.hpp:476-480: the raster plus the underlying pipeline run."""
    raster: Raster
    pipeline: PipelineOutcome


def run_raster(data: PointSet, nx: int, ny: int, cfg: RunConfig,
               with_alpha: bool = True) -> RasterOutcome:
    """The compute part of cli::cmd_raster (cli.hpp:484-524): the nx x ny
    lattice over bbox(data) is generated in HBM (no host lattice, no query
    upload), then the fused pipeline runs; host data in, raster out."""
    if nx < 1 or ny < 1:
        raise InvalidArgument("cmd_raster: nx and ny must be >= 1")
    if data.count() == 0:
        raise InvalidArgument("cmd_raster: data set is empty")
    n = nx * ny
    vals, alph, bb = np.empty(n), (np.empty(n) if with_alpha else None), np.empty(4)
    st = L.RunStats()
    c = cfg.c()
    err = L.Error()
    zs = data.zs if data.has_values() else None
    _raise(lib().aidw_run_raster(_p(data.xs), _p(data.ys), _p(zs) if zs is not None else None,
                                 data.count(), nx, ny, C.byref(c), _p(vals),
                                 _p(alph) if with_alpha else None, _p(bb),
                                 C.byref(st), C.byref(err)), err)
    raster = Raster(nx, ny, float(bb[0]), float(bb[1]), (bb[2] - bb[0]) / nx, vals)
    return RasterOutcome(raster, PipelineOutcome(InterpolationResult(vals, alph), st.as_dict(),
                                                 int(st.k_effective)))


def raster_lattice_device(nx, ny, bbox, d_xs, d_ys, row0=0, rows=None, stream=None):
    """cmd_raster lattice rows [row0, row0 + rows) generated into device
    buffers (raw pointers), cli.hpp:496-507."""
    rows = ny - row0 if rows is None else rows
    bb = _f64(bbox)
    err = L.Error()
    _raise(lib().aidw_raster_lattice_device(nx, ny, _p(bb), row0, rows, d_xs, d_ys, stream,
                                            C.byref(err)), err)


def write_raster_asc(path: str, raster: Raster) -> None:
    """io.hpp:199-221, byte-identical output, parallel formatting."""
    if len(raster.values) != raster.ncols * raster.nrows:
        raise InvalidArgument("write_raster_asc: value count does not match dimensions")
    v = _f64(raster.values)
    err = L.Error()
    _raise(lib().aidw_write_raster_asc(path.encode(), raster.ncols, raster.nrows,
                                       float(raster.xllcorner), float(raster.yllcorner),
                                       float(raster.cellsize), _p(v), C.byref(err)), err)


# ------------------------------------------------------------ files (io.hpp)
def _read_points(path, with_values):
    buf = L.PointsBuffer()
    err = L.Error()
    _raise(lib().aidw_read_points_csv(path.encode(), 1 if with_values else 0, C.byref(buf),
                                      C.byref(err)), err)
    try:
        n = buf.count
        xs = np.ctypeslib.as_array(buf.xs, (n,)).copy() if n else np.empty(0)
        ys = np.ctypeslib.as_array(buf.ys, (n,)).copy() if n else np.empty(0)
        zs = (np.ctypeslib.as_array(buf.zs, (n,)).copy() if n else np.empty(0)) \
            if with_values else np.empty(0)
    finally:
        lib().aidw_free_points(C.byref(buf))
    return PointSet(xs, ys, zs)


def read_data_csv(path: str) -> PointSet:
    """io.hpp:103-124: header `x,y,z`; parallel parse, reference diagnostics."""
    return _read_points(path, True)


def read_query_csv(path: str) -> PointSet:
    """io.hpp:126-145: header `x,y`."""
    return _read_points(path, False)


def _write_columns(path, header, cols):
    cols = [_f64(c) for c in cols]
    arr = (L._dp * len(cols))(*[_p(c) for c in cols])
    err = L.Error()
    _raise(lib().aidw_write_columns_csv(path.encode(), header.encode(), len(cols[0]), len(cols),
                                        arr, C.byref(err)), err)


def write_data_csv(path: str, data: PointSet) -> None:
    """io.hpp:146-156 ("%.17g" fields, byte-identical)."""
    if not data.has_values():
        raise InvalidArgument("write_data_csv: point set carries no values")
    _write_columns(path, "x,y,z", [data.xs, data.ys, data.zs])


def write_query_csv(path: str, queries: PointSet) -> None:
    """io.hpp:158-167."""
    _write_columns(path, "x,y", [queries.xs, queries.ys])


def write_result_csv(path: str, queries: PointSet, result: InterpolationResult) -> None:
    """io.hpp:169-188: `x,y,alpha,z_pred`, input order."""
    n = queries.count()
    if len(result.predicted) != n or len(result.alphas) != n:
        raise InvalidArgument("write_result_csv: result length does not match queries")
    _write_columns(path, "x,y,alpha,z_pred", [queries.xs, queries.ys, result.alphas,
                                              result.predicted])


def parse_raster_asc(path: str) -> Raster:
    """io.hpp:223-253."""
    buf = L.RasterBuffer()
    err = L.Error()
    _raise(lib().aidw_read_raster_asc(path.encode(), C.byref(buf), C.byref(err)), err)
    try:
        vals = np.ctypeslib.as_array(buf.values, (buf.count,)).copy() if buf.count else np.empty(0)
        return Raster(int(buf.ncols), int(buf.nrows), buf.xllcorner, buf.yllcorner, buf.cellsize,
                      vals)
    finally:
        lib().aidw_free_raster(C.byref(buf))


def compute_bbox_device(d_dx, d_dy, m, d_qx, d_qy, n, stream=None):
    out = np.empty(4)
    err = L.Error()
    _raise(lib().aidw_compute_bbox_device(d_dx, d_dy, m, d_qx, d_qy, n, _p(out), stream,
                                          C.byref(err)), err)
    return out
