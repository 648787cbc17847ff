"""At-scale parity: every BASELINE.json config at its full size, against the
reference itself (oracle/_ref/libaidw_ref.so, compiled in place from
/root/reference — test infrastructure only) and the C restatement.

SURVEY §8(d) "Parity set":
  * kNN in full at every config — here all 1M queries of configs[2]
    (uniform), configs[3] (clustered) and the clustered stress variant
    (uniform queries over blob data, expansion levels far beyond 2): d2
    lists, average distances and exhaustion bit-identical to the
    reference's knn_stage (knn.hpp:255-271), (d2, idx) index sets
    bit-identical to the C oracle's lexicographic lists;
  * predictions and alphas in full at 100K x 100K (configs[1]) against the
    reference's cli::run_pipeline (cli.hpp:217-268), FP32 (1e-5) and FP64
    (2e-11) weighting;
  * a stratified sample of a 1M x 1M run (snap, void, cluster-core and
    fractional-alpha queries) — the GPU interpolates all 1M queries, the
    reference the sample plus the queries that pin bbox(data ∪ queries), so
    both see the same grid, area and snap tolerance;
  * configs[4] (4M planar data, 4096^2 raster lattice, k = 15): kNN of all
    16.8M lattice queries against the reference's knn_stage; the full
    raster on the GPU (aidw_run_raster), >= 4096 lattice points spread over
    every row checked against the reference (the lattice lies inside
    bbox(data), so bbox, area and snap tolerance are the raster's).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu
UNIT = (0.0, 0.0, 1.0, 1.0)
FP32_TOL = 1e-5
FP64_TOL = 2e-11
THREADS = max(1, min(32, os.cpu_count() or 1))


def need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref/libaidw_ref.so not built (needs /root/reference at build time)")


def pred_err(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * span)))


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


@pytest.fixture(autouse=True)
def fp32_default():
    A.set_weight_precision("fp32")
    yield
    A.set_weight_precision("fp32")


def config_inputs(kind, n=1_000_000):
    """BASELINE configs[2] / [3] inputs and the stress
    variant: blob data with uniform queries (void queries widen many rings)."""
    m = 1_000_000
    if kind == "uniform":
        xs, ys, zs = O.generate_points(m, UNIT, 42)
        qx, qy = O.generate_queries(n, UNIT, 43)
    elif kind == "clustered":
        xs, ys, zs = O.generate_clustered(m, seed=42)
        qx, qy = O.generate_clustered(n, seed=43, with_values=False)
    else:
        xs, ys, zs = O.generate_clustered(m, seed=42)
        qx, qy = O.generate_queries(n, UNIT, 43)
    return xs, ys, zs, qx, qy


def oracle_knn_parallel(qx, qy, cfg, grid, m, k):
    parts = np.array_split(np.arange(qx.size), THREADS)
    with ThreadPoolExecutor(THREADS) as ex:  # ctypes drops the GIL per call
        res = list(ex.map(lambda p: O.knn_grid(qx[p], qy[p], cfg, grid, m, k), parts))
    return (np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res]),
            np.concatenate([r[2] for r in res]))


# ------------------------------------------------------------------ kNN, full
@pytest.mark.parametrize("kind", ["uniform", "clustered", "stress"])
def test_knn_stage_all_1m_queries(kind):
    need_ref()
    xs, ys, _, qx, qy = config_inputs(kind)
    m, k = xs.size, 10
    bb = O.compute_bbox(xs, ys, qx, qy)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(m, bb, 4.0))
    cfg = A.GridConfig(cfg_o.cell_width, cfg_o.n_col, cfg_o.n_row, cfg_o.min_x, cfg_o.min_y)
    index = A.build_index(A.PointSet(xs, ys), cfg)
    got = A.knn_stage(A.PointSet(qx, qy), index, A.PointSet(xs, ys), k)
    # the reference's own knn_stage (its grid over bbox(data ∪ queries), factor 4)
    ref_d2, ref_avg, ref_exh, ref_len = O.ref_knn_stage(qx, qy, xs, ys, k, factor=4.0,
                                                        workers=THREADS)
    assert np.all(ref_len == k) and not ref_exh.any() and not got.exhausted
    assert np.array_equal(got.distances_sq, ref_d2)
    assert np.array_equal(got.average_distance, ref_avg)
    # (d2, idx)-lexicographic index sets against the C restatement
    grid_o = O.build_index(xs, ys, cfg_o)
    assert np.array_equal(index.sorted_point_ids, grid_o[0])
    o_d2, o_ids, o_avg = oracle_knn_parallel(qx, qy, cfg_o, grid_o, m, k)
    assert np.array_equal(o_d2, ref_d2)
    assert np.array_equal(got.indices, o_ids)
    if kind == "stress":
        # the stress really stresses: many void queries need far more than the
        # reference's level-2 block (kth neighbour beyond 2 cell widths)
        far = np.sqrt(ref_d2[:, -1]) > 2.0 * cfg_o.cell_width
        assert far.mean() > 0.2


# ------------------------------------------------------------------ 100K full
@pytest.fixture(scope="module")
def ref_100k():
    need_ref()
    xs, ys, zs = O.generate_points(100_000, UNIT, 42)
    qx, qy = O.generate_queries(100_000, UNIT, 43)
    pred, alpha, _, keff = O.ref_run_pipeline(xs, ys, zs, qx, qy, mode=1, k=10, workers=THREADS)
    return xs, ys, zs, qx, qy, pred, alpha, keff


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_pipeline_100k_full(ref_100k, precision):
    """BASELINE configs[1] in full: every alpha and every prediction."""
    xs, ys, zs, qx, qy, ref_pred, ref_alpha, keff = ref_100k
    A.set_weight_precision(precision)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(params=A.AidwParams(k=10)))
    assert out.k_effective == keff == 10
    sat = ref_alpha == 4.0
    assert sat.mean() > 0.9
    assert np.array_equal(out.result.alphas[sat], ref_alpha[sat])
    assert rel_err(out.result.alphas, ref_alpha) <= 1e-12
    tol = FP32_TOL if precision == "fp32" else FP64_TOL
    assert pred_err(out.result.predicted, ref_pred, zs) <= tol


# ------------------------------------------------------------------ 1M stratified
def stratified_queries(xs, ys, seed=7):
    """1M queries over 1M blob points: uniform (voids), blob-distributed,
    cluster-core (the densest histogram bins), and snap queries (data sites,
    exactly and within the snap tolerance).  Returns (qx, qy, strata) with
    strata[name] = query indices."""
    rng = np.random.default_rng(seed)
    n_uni, n_core, n_snap = 450_000, 40_000, 10_000
    ux, uy = O.generate_queries(n_uni, UNIT, 43)
    bx, by = O.generate_clustered(1_000_000 - n_uni - n_core - n_snap, seed=44, with_values=False)
    h, ex, ey = np.histogram2d(xs, ys, bins=64, range=[[0, 1], [0, 1]])
    dense = np.argsort(h.ravel())[-16:]
    b = rng.choice(dense, n_core)
    cx = ex[b // 64] + rng.random(n_core) / 64
    cy = ey[b % 64] + rng.random(n_core) / 64
    sites = rng.choice(xs.size, n_snap, replace=False)
    sx, sy = xs[sites].copy(), ys[sites].copy()
    diag = np.hypot(1.0, 1.0)
    sx[n_snap // 2:] += 0.3e-12 * diag  # inside (1e-12 diag)^2 (interpolate.hpp:86-89)
    qx = np.concatenate([ux, bx, cx, sx])
    qy = np.concatenate([uy, by, cy, sy])
    perm = rng.permutation(qx.size)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    qx, qy = qx[perm], qy[perm]
    o_uni, o_blob = 0, n_uni
    o_core = o_blob + bx.size
    o_snap = o_core + n_core
    strata = {"uniform": inv[o_uni:o_blob], "blob": inv[o_blob:o_core],
              "core": inv[o_core:o_snap], "snap": inv[o_snap:]}
    return qx, qy, strata


def test_pipeline_1m_stratified_sample():
    need_ref()
    xs, ys, zs = O.generate_clustered(1_000_000, seed=42)
    qx, qy, strata = stratified_queries(xs, ys)
    data, q = A.PointSet(xs, ys, zs), A.PointSet(qx, qy)
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    alpha = out.result.alphas
    rng = np.random.default_rng(11)
    pick = []
    # void queries: uniform queries with alpha at the top level (far from blobs)
    void = strata["uniform"][alpha[strata["uniform"]] == 4.0]
    frac = strata["blob"][(alpha[strata["blob"]] % 0.5) != 0.0]  # fractional alpha (lerp)
    core = strata["core"]
    snap = strata["snap"]
    for pool in (void, frac, core, snap):
        assert pool.size >= 1024
        pick.append(rng.choice(pool, 1024, replace=False))
    # the queries that pin bbox(data ∪ queries): same grid, area, snap tolerance
    pick.append(np.array([np.argmin(qx), np.argmax(qx), np.argmin(qy), np.argmax(qy)]))
    s = np.unique(np.concatenate(pick))
    bb_all = O.compute_bbox(xs, ys, qx, qy)
    assert np.array_equal(O.compute_bbox(xs, ys, qx[s], qy[s]), bb_all)
    ref_pred, ref_alpha, _, _ = O.ref_run_pipeline(xs, ys, zs, qx[s], qy[s], mode=1, k=10,
                                                   workers=THREADS)
    assert rel_err(alpha[s], ref_alpha) <= 1e-12
    in_core = np.isin(s, core)
    assert np.median(ref_alpha[in_core]) < 1.5  # dense cores: low alpha (adaptive.hpp:69-87)
    assert pred_err(out.result.predicted[s], ref_pred, zs) <= FP32_TOL
    snapped = np.isin(s, snap)
    assert np.array_equal(out.result.predicted[s][snapped], ref_pred[snapped])
    A.set_weight_precision("fp64")
    out64 = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    assert np.array_equal(out64.result.alphas, alpha)
    assert rel_err(out64.result.predicted[s], ref_pred) <= FP64_TOL


# ------------------------------------------------------------------ IDW at scale
@pytest.mark.parametrize("alpha", [2.0, 2.5])
def test_idw_1m_sample(alpha):
    """Constant-alpha IDW over 1M points (idw_predict_all, interpolate.hpp:426-448;
    alpha = 2: the reference's default exponent, one tensor-core recipe
    class; 2.5: the general form on the CUDA cores): all 1M queries on the
    GPU, 4096 of them spread over the index range against the reference's
    run_pipeline in idw mode, plus the bbox-pinning queries."""
    need_ref()
    xs, ys, zs = O.generate_points(1_000_000, UNIT, 42)
    qx, qy = O.generate_queries(1_000_000, UNIT, 43)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(mode="idw", alpha=alpha))
    s = np.unique(np.concatenate([np.arange(0, qx.size, qx.size // 4096),
                                  [np.argmin(qx), np.argmax(qx), np.argmin(qy), np.argmax(qy)]]))
    assert np.array_equal(O.compute_bbox(xs, ys, qx[s], qy[s]), O.compute_bbox(xs, ys, qx, qy))
    ref_pred, _, _, _ = O.ref_run_pipeline(xs, ys, zs, qx[s], qy[s], mode=0, alpha=alpha,
                                           workers=THREADS)
    assert pred_err(out.result.predicted[s], ref_pred, zs) <= FP32_TOL
    assert np.all(out.result.alphas == alpha)


# ------------------------------------------------------------------ DEM kNN, full
def test_dem_knn_stage_all_lattice_queries():
    """configs[4] kNN in full: all 4096^2 lattice queries over 4M planar
    points, k = 15 — d2 lists and averages bit-identical to the reference's
    knn_stage (knn.hpp:255-271); (d2, idx) index sets against the C oracle on
    every 16th lattice row (the oracle is single-pass C: bounded time)."""
    need_ref()
    nx = ny = 4096
    k = 15
    xs, ys, _ = O.generate_points(4_000_000, UNIT, 42, 1)
    bb = O.compute_bbox(xs, ys)
    qx, qy = O.raster_lattice(nx, ny, bb)
    assert np.array_equal(O.compute_bbox(xs, ys, qx, qy), bb)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, 4.0))
    cfg = A.GridConfig(cfg_o.cell_width, cfg_o.n_col, cfg_o.n_row, cfg_o.min_x, cfg_o.min_y)
    index = A.build_index(A.PointSet(xs, ys), cfg)
    got = A.knn_stage(A.PointSet(qx, qy), index, A.PointSet(xs, ys), k)
    ref_d2, ref_avg, ref_exh, ref_len = O.ref_knn_stage(qx, qy, xs, ys, k, factor=4.0,
                                                        workers=THREADS)
    assert np.all(ref_len == k) and not ref_exh.any() and not got.exhausted
    assert np.array_equal(got.distances_sq, ref_d2)
    assert np.array_equal(got.average_distance, ref_avg)
    del ref_d2, ref_avg
    grid_o = O.build_index(xs, ys, cfg_o)
    assert np.array_equal(index.sorted_point_ids, grid_o[0])
    rows = np.arange(0, ny, 16)
    sel = (rows[:, None] * nx + np.arange(nx)[None, :]).ravel()
    o_d2, o_ids, _ = oracle_knn_parallel(qx[sel], qy[sel], cfg_o, grid_o, xs.size, k)
    assert np.array_equal(got.distances_sq[sel], o_d2)
    assert np.array_equal(got.indices[sel], o_ids)


# ------------------------------------------------------------------ DEM raster
def test_dem_raster_sample():
    """configs[4]: 4M planar points, 4096 x 4096 lattice, k = 15."""
    need_ref()
    nx = ny = 4096
    xs, ys, zs = O.generate_points(4_000_000, UNIT, 42, 1)
    out = A.run_raster(A.PointSet(xs, ys, zs), nx, ny, A.RunConfig(params=A.AidwParams(k=15)))
    vals, alpha = out.raster.values, out.pipeline.result.alphas
    assert vals.size == nx * ny and np.all(np.isfinite(vals))
    bb = O.compute_bbox(xs, ys)
    assert (out.raster.xllcorner, out.raster.yllcorner) == (bb[0], bb[1])
    lx, ly = O.raster_lattice(nx, ny, bb)
    # two lattice points per row, columns spread by a hash: 8192 points
    rows = np.repeat(np.arange(ny), 2)
    cols = (rows * 2654435761 + np.tile([0, nx // 2], ny) * 7919) % nx
    s = rows * nx + cols
    ref_pred, ref_alpha, _, keff = O.ref_run_pipeline(xs, ys, zs, lx[s], ly[s], mode=1, k=15,
                                                      workers=THREADS)
    assert keff == 15
    assert rel_err(alpha[s], ref_alpha) <= 1e-12
    assert pred_err(vals[s], ref_pred, zs) <= FP32_TOL
    # planar value rule: the interpolated surface is within 5 % of the plane
    # (test_cli.cpp:266-309's raster check, on the interior)
    truth = 1.5 * lx[s] - 2.5 * ly[s] + 4.0
    inner = (lx[s] > 0.05) & (lx[s] < 0.95) & (ly[s] > 0.05) & (ly[s] < 0.95)
    assert np.max(np.abs(vals[s][inner] - truth[inner]) / np.abs(truth[inner])) <= 0.05
