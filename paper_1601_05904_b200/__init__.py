"""B200-native AIDW (adaptive inverse distance weighting) with even-grid kNN.

Drop-in for the reference's AIDW hot path (proj/include/aidw): grid build
(K1), exact grid kNN + adaptive alpha (K2 + K3) and the O(m·n) weighting
(K4), each a hand-written sm_100a kernel in csrc/, exposed through the C-ABI
include/aidw_capi.h.  This package is the Python host mirror of the
reference API over that C-ABI (api.py) plus the ctypes binding (_lib.py).
"""
from .api import (  # noqa: F401
    AidwParams, AidwRuntimeError, BoundingBox, CudaError, DomainError, GridConfig, GridIndex,
    InterpolationResult, InvalidArgument, KnnStageResult, OutOfRange, PipelineOutcome, PointSet,
    Raster, RasterOutcome, RunConfig, aidw_predict_all, build_index, choose_cell_width,
    compute_bbox, compute_bbox_device, graph_counters, set_graphs, device_count, device_info, generate_clustered, generate_random_points,
    generate_random_queries, idw_predict_all, kernel_launch_count, knn_stage, make_grid_config,
    parse_raster_asc, raster_lattice, replication_info, raster_lattice_device, read_data_csv, read_query_csv,
    run_pipeline, run_pipeline_device, run_raster, set_alpha4_recipe, set_devices, set_query_slab, weight_engine,
    set_weight_precision,
    write_data_csv, write_query_csv, write_raster_asc, write_result_csv)

__version__ = "0.1.0"
