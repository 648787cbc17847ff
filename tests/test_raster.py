"""cmd_raster path: the lattice generated in HBM, the
raster run (aidw_run_raster) and the ASCII-grid writer.

Oracles: the C restatement of the lattice (oracle/aidw_oracle.c,
cli.hpp:495-507), and the reference itself — cli::cmd_raster through
oracle/_ref (CSV writer/parser, run_pipeline, write_raster_asc), whose .asc
output pins the writer byte for byte."""
import os

import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

UNIT = (0.0, 0.0, 1.0, 1.0)


def fmt(v):
    return "%.17g" % v


def asc_text(ncols, nrows, xll, yll, cell, values):
    lines = [f"ncols {ncols}", f"nrows {nrows}", f"xllcorner {fmt(xll)}",
             f"yllcorner {fmt(yll)}", f"cellsize {fmt(cell)}"]
    for r in range(nrows):
        lines.append(" ".join(fmt(v) for v in values[r * ncols:(r + 1) * ncols]))
    return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ CPU
def test_writer_matches_printf(tmp_path):  # io.hpp:25-29 ("%.17g"), :199-221
    rng = np.random.default_rng(3)
    v = rng.standard_normal(700) * 10.0 ** rng.integers(-300, 300, 700)
    v[:9] = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3]
    r = A.Raster(35, 20, 0.123456789, -5.5, 1 / 3, v)
    path = str(tmp_path / "r.asc")
    A.write_raster_asc(path, r)
    assert open(path).read() == asc_text(35, 20, 0.123456789, -5.5, 1 / 3, v)


def test_writer_large_parallel(tmp_path):  # many rows across the thread batches
    v = np.arange(3000 * 41, dtype=np.float64) / 7.0
    r = A.Raster(41, 3000, 0.0, 0.0, 1.0, v)
    path = str(tmp_path / "big.asc")
    A.write_raster_asc(path, r)
    assert open(path).read() == asc_text(41, 3000, 0.0, 0.0, 1.0, v)


def test_writer_errors(tmp_path):
    with pytest.raises(A.InvalidArgument, match="value count does not match"):
        A.write_raster_asc(str(tmp_path / "x.asc"), A.Raster(3, 2, 0.0, 0.0, 1.0, np.zeros(5)))
    with pytest.raises(A.AidwRuntimeError, match="cannot open for writing"):
        A.write_raster_asc(str(tmp_path / "no" / "such" / "dir.asc"),
                           A.Raster(1, 1, 0.0, 0.0, 1.0, np.zeros(1)))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_writer_byte_identical_to_reference(tmp_path):
    """The reference's cmd_raster writes its raster with write_raster_asc; the
    same raster through our writer must give the same bytes."""
    dx, dy, dz = O.generate_points(3000, UNIT, 42, 1)
    vals, meta, asc = O.ref_cmd_raster(dx, dy, dz, 23, 17, k=10, tmpdir=str(tmp_path))
    ours = str(tmp_path / "ours.asc")
    A.write_raster_asc(ours, A.Raster(int(meta["ncols"]), int(meta["nrows"]), meta["xllcorner"],
                                      meta["yllcorner"], meta["cellsize"], vals))
    assert open(ours, "rb").read() == open(asc, "rb").read()


def test_host_lattice_matches_oracle():
    for nx, ny, bb in [(3, 2, (0.0, 0.0, 3.0, 2.0)), (17, 5, (-1.5, 2.25, 7.0, 3.0)),
                       (64, 64, (0.1, 0.2, 0.9, 0.7))]:
        xo, yo = O.raster_lattice(nx, ny, bb)
        lat = A.raster_lattice(nx, ny, bb)
        assert np.array_equal(lat.xs, xo) and np.array_equal(lat.ys, yo)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,row0,rows,bb", [
    (3, 2, 0, 2, (0.0, 0.0, 3.0, 2.0)),
    (257, 131, 0, 131, (-3.25, 1e-3, 11.0, 0.9)),
    (1000, 700, 123, 301, (0.123, 0.456, 0.789, 1.012)),  # a shard of rows
])
def test_device_lattice_bit_exact(nx, ny, row0, rows, bb):  # cli.hpp:495-507
    import torch
    xs = torch.empty(nx * rows, dtype=torch.float64, device="cuda")
    ys = torch.empty_like(xs)
    A.raster_lattice_device(nx, ny, bb, xs.data_ptr(), ys.data_ptr(), row0, rows)
    torch.cuda.synchronize()
    xo, yo = O.raster_lattice(nx, ny, bb)
    sl = slice(row0 * nx, (row0 + rows) * nx)
    assert np.array_equal(xs.cpu().numpy(), xo[sl])
    assert np.array_equal(ys.cpu().numpy(), yo[sl])


@pytest.mark.gpu
def test_run_raster_equals_pipeline_on_host_lattice():
    data = A.generate_random_points(20_000, UNIT, 7, "planar")
    out = A.run_raster(data, 96, 80, A.RunConfig(params=A.AidwParams(k=15)))
    bb = A.compute_bbox(data)
    lat = A.raster_lattice(96, 80, (bb.min_x, bb.min_y, bb.max_x, bb.max_y))
    ref = A.run_pipeline(data, lat, A.RunConfig(params=A.AidwParams(k=15)))
    assert np.array_equal(out.raster.values, ref.result.predicted)
    assert np.array_equal(out.pipeline.result.alphas, ref.result.alphas)
    assert out.raster.grid().shape == (80, 96)
    assert out.raster.xllcorner == bb.min_x and out.raster.yllcorner == bb.min_y
    assert out.raster.cellsize == (bb.max_x - bb.min_x) / 96


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_run_raster_vs_reference_cmd_raster(tmp_path):
    """The reference's cli::cmd_raster end to end (CSV in, .asc out) against
    run_raster + write_raster_asc: header lines identical, values within the
    FP32 contract (and within 2e-11 in FP64 mode)."""
    dx, dy, dz = O.generate_points(5000, UNIT, 42, 1)
    vals, meta, asc = O.ref_cmd_raster(dx, dy, dz, 48, 36, k=15, tmpdir=str(tmp_path))
    data = A.PointSet(dx, dy, dz)
    out = A.run_raster(data, 48, 36, A.RunConfig(params=A.AidwParams(k=15)))
    span = dz.max() - dz.min()
    err = np.max(np.abs(out.raster.values - vals) / np.maximum(np.abs(vals), 1e-3 * span))
    assert err <= 1e-5, err
    ours = str(tmp_path / "ours.asc")
    A.write_raster_asc(ours, out.raster)
    head_ref = open(asc).read().splitlines()[:5]
    head_ours = open(ours).read().splitlines()[:5]
    assert head_ours == head_ref
    A.set_weight_precision("fp64")
    try:
        out64 = A.run_raster(data, 48, 36, A.RunConfig(params=A.AidwParams(k=15)))
    finally:
        A.set_weight_precision("fp32")
    assert np.max(np.abs(out64.raster.values - vals) / np.abs(vals)) <= 2e-11


@pytest.mark.gpu
def test_run_raster_errors():
    data = A.generate_random_points(100, UNIT, 1)
    with pytest.raises(A.InvalidArgument, match="nx and ny must be >= 1"):
        A.run_raster(data, 0, 5, A.RunConfig())
    with pytest.raises(A.InvalidArgument, match="data set is empty"):
        A.run_raster(A.PointSet(np.empty(0), np.empty(0), np.empty(0)), 4, 4, A.RunConfig())
