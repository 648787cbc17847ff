"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/aidw_capi.h declares, the Python mirror binds them all,
host-only entry points (generators) agree with the oracle bit-for-bit, and
compute entry points fail loudly (AIDW_ERR_CUDA) when no GPU is present."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1601_05904_b200 import _lib as L
import paper_1601_05904_b200 as A


def test_library_exports_every_header_symbol():
    lib = L.load()
    declared = L.header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(L.SIGNATURES), "Python binding out of sync with the header"
    assert lib.aidw_capi_version() == 1


def test_generators_match_oracle():
    for rule in ("uniform", "planar", "radial"):
        p = A.generate_random_points(3000, (-3.0, 5.0, 17.0, 25.0), 1003, rule)
        xs, ys, zs = O.generate_points(3000, (-3.0, 5.0, 17.0, 25.0), 1003,
                                       {"uniform": 0, "planar": 1, "radial": 2}[rule])
        assert np.array_equal(p.xs, xs) and np.array_equal(p.ys, ys) and np.array_equal(p.zs, zs)
    q = A.generate_random_queries(2000, (0, 0, 1, 1), 43)
    qx, qy = O.generate_queries(2000, (0, 0, 1, 1), 43)
    assert np.array_equal(q.xs, qx) and np.array_equal(q.ys, qy)
    c = A.generate_clustered(5000, seed=42)
    cx, cy, cz = O.generate_clustered(5000, seed=42)
    assert np.array_equal(c.xs, cx) and np.array_equal(c.zs, cz)


def test_raster_lattice_north_first():  # cli.hpp:496-507
    r = A.raster_lattice(3, 2, (0.0, 0.0, 3.0, 2.0))
    assert r.xs.tolist() == [0.5, 1.5, 2.5, 0.5, 1.5, 2.5]
    assert r.ys.tolist() == [1.5, 1.5, 1.5, 0.5, 0.5, 0.5]


def test_generator_errors():
    with pytest.raises(A.InvalidArgument):
        A.generate_random_points(0)
    with pytest.raises(A.InvalidArgument):
        A.generate_random_queries(10, (0.0, 0.0, 0.0, 1.0))


def test_host_setup_helpers_match_oracle():
    data = A.generate_random_points(1000, (0, 0, 1, 1), 42)
    q = A.generate_random_queries(100, (0, 0, 1, 1), 43)
    bb = A.compute_bbox(data, q)
    ob = O.compute_bbox(data.xs, data.ys, q.xs, q.ys)
    assert bb.as_array().tolist() == ob.tolist()
    w = A.choose_cell_width(data, bb, 4.0)
    assert w == O.choose_cell_width(1000, ob, 4.0)
    cfg, ocfg = A.make_grid_config(bb, w), O.make_grid_config(ob, w)
    assert (cfg.n_col, cfg.n_row, cfg.cell_width) == (ocfg.n_col, ocfg.n_row, ocfg.cell_width)
    with pytest.raises(A.InvalidArgument):
        A.make_grid_config(A.BoundingBox(0, 0, 1, 1), 1e-9)


def test_compute_paths_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    data = A.generate_random_points(100, (0, 0, 1, 1), 1)
    q = A.generate_random_queries(10, (0, 0, 1, 1), 2)
    with pytest.raises(A.CudaError):
        A.run_pipeline(data, q, A.RunConfig())
    with pytest.raises(A.CudaError):
        A.build_index(data, A.GridConfig(0.25, 5, 5, 0.0, 0.0))
