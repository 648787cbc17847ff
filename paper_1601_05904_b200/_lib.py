"""ctypes binding of libaidw_b200.so (include/aidw_capi.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_1601_05904_b200/csrc``.  Loading fails loudly when it is
missing: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# AIDW_LIB_PATH: an alternative build of the same library (kernel-tuning
# experiments); the default is the in-tree build
LIB_PATH = os.environ.get("AIDW_LIB_PATH") or os.path.join(HERE, "lib", "libaidw_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "aidw_capi.h")

AIDW_OK = 0
AIDW_ERR_INVALID_ARGUMENT = 1
AIDW_ERR_DOMAIN = 2
AIDW_ERR_OUT_OF_RANGE = 3
AIDW_ERR_RUNTIME = 4
AIDW_ERR_CUDA = 5

ENGINE_GRID, ENGINE_BRUTE = 0, 1
VARIANT_NAIVE, VARIANT_BLOCKED = 0, 1
MODE_IDW, MODE_AIDW = 0, 1
PRECISION_FP32, PRECISION_FP64 = 0, 1


class Error(C.Structure):
    _fields_ = [("code", C.c_int32), ("index", C.c_int64), ("message", C.c_char * 512)]


class GridConfig(C.Structure):
    _fields_ = [("cell_width", C.c_double), ("n_col", C.c_int32), ("n_row", C.c_int32),
                ("min_x", C.c_double), ("min_y", C.c_double)]

    def cell_total(self):
        return int(self.n_col) * int(self.n_row)


class Params(C.Structure):
    _fields_ = [("k", C.c_int32), ("r_min", C.c_double), ("r_max", C.c_double),
                ("alpha_levels", C.c_double * 5), ("area", C.c_double)]


class RunConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("engine", C.c_int32), ("variant", C.c_int32),
                ("params", Params), ("alpha", C.c_double), ("cell_factor", C.c_double),
                ("workers", C.c_int32), ("use_bbox", C.c_int32), ("bbox", C.c_double * 4)]


class RunStats(C.Structure):
    _fields_ = [("build_ms", C.c_double), ("knn_ms", C.c_double), ("interp_ms", C.c_double),
                ("total_ms", C.c_double), ("weight_kernel_ms", C.c_double),
                ("knn_kernel_ms", C.c_double), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double),
                ("k_effective", C.c_int32), ("worker_count", C.c_int32), ("pairs", C.c_int64),
                ("knn_candidates", C.c_int64), ("knn_ref_candidates", C.c_int64),
                ("alpha4_queries", C.c_int64),
                ("kernel_launches", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_ep = C.POINTER(Error)

class PointsBuffer(C.Structure):
    _fields_ = [("xs", C.POINTER(C.c_double)), ("ys", C.POINTER(C.c_double)),
                ("zs", C.POINTER(C.c_double)), ("count", C.c_size_t)]


class RasterBuffer(C.Structure):
    _fields_ = [("ncols", C.c_size_t), ("nrows", C.c_size_t), ("xllcorner", C.c_double),
                ("yllcorner", C.c_double), ("cellsize", C.c_double),
                ("values", C.POINTER(C.c_double)), ("count", C.c_size_t)]


# name -> (restype, argtypes); every symbol declared in include/aidw_capi.h
SIGNATURES = {
    "aidw_capi_version": (C.c_int, []),
    "aidw_kernel_launch_count": (C.c_int64, []),
    "aidw_device_info": (C.c_int, [C.c_char_p, C.c_size_t, _i32p, _ep]),
    "aidw_set_weight_precision": (None, [C.c_int32]),
    "aidw_get_weight_precision": (C.c_int32, []),
    "aidw_set_alpha4_recipe": (None, [C.c_int32]),
    "aidw_set_query_slab": (None, [C.c_int64]),
    "aidw_weight_engine": (C.c_int32, [C.c_int64]),
    "aidw_set_devices": (C.c_int, [_i32p, C.c_int32, _ep]),
    "aidw_device_count": (C.c_int32, []),
    "aidw_nccl_broadcast_count": (C.c_int64, []),
    "aidw_graph_counters": (None, [_i64p, _i64p]),
    "aidw_set_graphs": (None, [C.c_int32]),
    "aidw_last_replication": (C.c_int32, []),
    "aidw_nccl_version": (C.c_int32, []),
    "aidw_build_index": (C.c_int, [_dp, _dp, C.c_size_t, C.POINTER(GridConfig), _u32p, _u32p,
                                   _dp, _dp, _ep]),
    "aidw_build_index_mirror": (C.c_int, [_dp, _dp, C.c_size_t, C.POINTER(GridConfig), _u32p,
                                          _u32p, _dp, _dp, C.POINTER(C.c_void_p), _ep]),
    "aidw_index_release": (None, [C.c_void_p]),
    "aidw_index_info": (C.c_int, [C.c_void_p, C.POINTER(GridConfig), C.POINTER(C.c_size_t)]),
    "aidw_pinned_alloc": (C.c_void_p, [C.c_size_t]),
    "aidw_pinned_free": (None, [C.c_void_p]),
    "aidw_knn_stage_mirror": (C.c_int, [_dp, _dp, C.c_size_t, C.c_void_p, C.c_int32, _dp, _u32p,
                                        _dp, _i32p, _i32p, _ep]),
    "aidw_knn_stage": (C.c_int, [_dp, _dp, C.c_size_t, C.POINTER(GridConfig), _u32p, _u32p,
                                 _dp, _dp, _dp, _dp, C.c_size_t, C.c_int32, C.c_int32, _dp,
                                 _u32p, _dp, _i32p, _i32p, _ep]),
    "aidw_aidw_predict_all": (C.c_int, [_dp, _dp, C.c_size_t, _dp, _dp, _dp, C.c_size_t, _dp,
                                        _i64p, _u8p, C.POINTER(Params), C.c_int32, C.c_int32,
                                        _dp, _dp, _ep]),
    "aidw_idw_predict_all": (C.c_int, [_dp, _dp, C.c_size_t, _dp, _dp, _dp, C.c_size_t,
                                       C.c_double, C.c_int32, C.c_int32, _dp, _dp, _ep]),
    "aidw_run_pipeline": (C.c_int, [_dp, _dp, _dp, C.c_size_t, _dp, _dp, C.c_size_t,
                                    C.POINTER(RunConfig), _dp, _dp, C.POINTER(RunStats), _ep]),
    "aidw_run_pipeline_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                           C.c_void_p, C.c_void_p, C.c_size_t,
                                           C.POINTER(RunConfig), C.c_void_p, C.c_void_p,
                                           C.POINTER(RunStats), C.c_void_p, _ep]),
    "aidw_compute_bbox_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                           C.c_void_p, C.c_size_t, _dp, C.c_void_p, _ep]),
    "aidw_generate_points": (C.c_int, [C.c_size_t, _dp, C.c_uint64, C.c_int32, _dp, _dp, _dp,
                                       _ep]),
    "aidw_generate_queries": (C.c_int, [C.c_size_t, _dp, C.c_uint64, _dp, _dp, _ep]),
    "aidw_generate_clustered": (C.c_int, [C.c_size_t, C.c_int32, C.c_double, C.c_uint64,
                                          C.c_uint64, _dp, _dp, _dp, _ep]),
    "aidw_raster_lattice": (C.c_int, [C.c_size_t, C.c_size_t, _dp, _dp, _dp, _ep]),
    "aidw_raster_lattice_device": (C.c_int, [C.c_size_t, C.c_size_t, _dp, C.c_size_t,
                                             C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                             _ep]),
    "aidw_run_raster": (C.c_int, [_dp, _dp, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                  C.POINTER(RunConfig), _dp, _dp, _dp, C.POINTER(RunStats),
                                  _ep]),
    "aidw_write_raster_asc": (C.c_int, [C.c_char_p, C.c_size_t, C.c_size_t, C.c_double,
                                        C.c_double, C.c_double, _dp, _ep]),
    "aidw_read_points_csv": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(PointsBuffer), _ep]),
    "aidw_free_points": (None, [C.POINTER(PointsBuffer)]),
    "aidw_write_columns_csv": (C.c_int, [C.c_char_p, C.c_char_p, C.c_size_t, C.c_int32,
                                         C.POINTER(_dp), _ep]),
    "aidw_read_raster_asc": (C.c_int, [C.c_char_p, C.POINTER(RasterBuffer), _ep]),
    "aidw_free_raster": (None, [C.POINTER(RasterBuffer)]),
}

_lib = None


def load():
    """Load libaidw_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing — build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def header_symbols(path=HEADER_PATH):
    """Function names declared in include/aidw_capi.h."""
    import re
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|void)\s*\*?\s*(aidw_\w+)\s*\(", text,
                                 flags=re.M)))
