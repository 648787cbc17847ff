"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference's golden fixtures.  Bar:

  * grid arrays, kNN squared-distance lists, average distances: bit-exact;
  * kNN index sets: (d2, idx)-lexicographic, bit-exact vs the C oracle;
  * alpha: bit-exact where mu saturates, else <= 1e-12 relative (device cos
    vs glibc cos);
  * predictions, FP32 K4: |gpu - ref| <= 1e-5 * max(|ref|, 1e-3 * hull span);
  * predictions, FP64 kernel: <= 2e-11 * max(1, m / 1e6) relative.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
UNIT = (0.0, 0.0, 1.0, 1.0)
FP32_TOL = 1e-5
FP64_TOL = 2e-11


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def pred_err(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    den = np.maximum(np.abs(ref), 1e-3 * span)
    return float(np.max(np.abs(got - ref) / den))


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


@pytest.fixture(autouse=True)
def fp32_default():
    A.set_weight_precision("fp32")
    yield
    A.set_weight_precision("fp32")


# ------------------------------------------------------------------ K1
@pytest.mark.parametrize("tag", ["a", "b"])
def test_build_index_golden(tag):
    g = gold("grid")
    c = g[f"{tag}_cfg"]
    cfg = A.GridConfig(c[0], int(c[1]), int(c[2]), c[3], c[4])
    idx = A.build_index(A.PointSet(g[f"{tag}_x"], g[f"{tag}_y"]), cfg)
    assert np.array_equal(idx.sorted_point_ids, g[f"{tag}_ids"])
    assert np.array_equal(idx.cell_start, g[f"{tag}_cell_start"])
    assert np.array_equal(idx.sorted_x, g[f"{tag}_sx"])
    assert np.array_equal(idx.sorted_y, g[f"{tag}_sy"])


@pytest.mark.parametrize("m,factor,gen", [(100_000, 4.0, "uniform"), (300_000, 1.0, "uniform"),
                                          (200_000, 4.0, "clustered"), (1, 4.0, "uniform"),
                                          (5000, 64.0, "uniform")])
def test_build_index_vs_oracle(m, factor, gen):
    if gen == "clustered":
        xs, ys, _ = O.generate_clustered(m, seed=11)
    else:
        xs, ys, _ = O.generate_points(m, UNIT, 11)
    bb = np.array(UNIT)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(m, bb, factor))
    ids, cs, sx, sy = O.build_index(xs, ys, cfg_o)
    cfg = A.GridConfig(cfg_o.cell_width, cfg_o.n_col, cfg_o.n_row, cfg_o.min_x, cfg_o.min_y)
    g = A.build_index(A.PointSet(xs, ys), cfg)
    assert np.array_equal(g.sorted_point_ids, ids)
    assert np.array_equal(g.cell_start, cs)
    assert np.array_equal(g.sorted_x, sx) and np.array_equal(g.sorted_y, sy)


@pytest.mark.parametrize("dups,cells_wide", [(20, 4.0), (200, 4.0), (300, 4.0), (5000, 4.0), (9000, 64.0)])
def test_build_index_crowded_cells(dups, cells_wide):
    """Every per-cell sort path of the counting-sort build: thread per cell
    (<= 16 points), CTA bitonic (17..4096), stable compaction (> 4096) —
    duplicates of one point plus a jittered cluster, interleaved by index."""
    rng = np.random.default_rng(dups)
    bx, by, _ = O.generate_points(3000, UNIT, 5)
    cx = np.full(dups, 0.5) + rng.integers(0, 3, dups) * 1e-9
    cy = np.full(dups, 0.25)
    xs = np.empty(3000 + dups)
    ys = np.empty(3000 + dups)
    order = rng.permutation(3000 + dups)
    xs[order] = np.concatenate([bx, cx])
    ys[order] = np.concatenate([by, cy])
    bb = np.array(UNIT)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, cells_wide))
    ids, cs, sx, sy = O.build_index(xs, ys, cfg_o)
    cfg = A.GridConfig(cfg_o.cell_width, cfg_o.n_col, cfg_o.n_row, cfg_o.min_x, cfg_o.min_y)
    g = A.build_index(A.PointSet(xs, ys), cfg)
    assert np.max(np.diff(cs)) >= dups
    assert np.array_equal(g.sorted_point_ids, ids)
    assert np.array_equal(g.cell_start, cs)
    assert np.array_equal(g.sorted_x, sx) and np.array_equal(g.sorted_y, sy)


def test_build_index_2x2_and_errors():  # test_grid.cpp:150-170, :276-279
    g = A.build_index(A.PointSet([1.5, 0.5, 1.5, 0.5], [0.5, 1.5, 1.5, 0.5]),
                      A.GridConfig(1.0, 2, 2, 0.0, 0.0))
    assert g.sorted_point_ids.tolist() == [3, 0, 1, 2]
    with pytest.raises(A.InvalidArgument):
        A.build_index(A.PointSet(), A.GridConfig(1.0, 1, 1, 0.0, 0.0))
    with pytest.raises(A.DomainError) as e:
        A.build_index(A.PointSet([0.5, 9.0], [0.5, 0.5]), A.GridConfig(1.0, 2, 2, 0.0, 0.0))
    assert e.value.index == 1 and "outside the covered region" in str(e.value)


# ------------------------------------------------------------------ K2
def _grid_for(xs, ys, qx, qy, factor):
    bb = O.compute_bbox(xs, ys, qx, qy)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, factor))
    cfg = A.GridConfig(cfg_o.cell_width, cfg_o.n_col, cfg_o.n_row, cfg_o.min_x, cfg_o.min_y)
    return cfg_o, A.build_index(A.PointSet(xs, ys), cfg)


@pytest.mark.parametrize("tag", ["std", "tiny", "exh"])
def test_knn_golden(tag):
    g = gold("knn")
    xs, ys, qx, qy = g[f"{tag}_x"], g[f"{tag}_y"], g[f"{tag}_qx"], g[f"{tag}_qy"]
    _, index = _grid_for(xs, ys, qx, qy, float(g[f"{tag}_factor"][0]))
    for k in g[f"{tag}_ks"]:
        k = int(k)
        r = A.knn_stage(A.PointSet(qx, qy), index, A.PointSet(xs, ys), k)
        ref = g[f"{tag}_k{k}_d2"]
        assert np.array_equal(r.distances_sq, ref[:, :r.k_effective])
        assert np.array_equal(r.average_distance, g[f"{tag}_k{k}_avg"])
        assert r.exhausted == bool(g[f"{tag}_k{k}_exh"][0])
        if k <= xs.size:
            bd2, bids, _ = O.knn_brute(qx, qy, xs, ys, k)
            assert np.array_equal(r.indices, bids)
            b = A.knn_stage(A.PointSet(qx, qy), None, A.PointSet(xs, ys), k, engine="brute")
            assert np.array_equal(b.distances_sq, r.distances_sq)
            assert np.array_equal(b.indices, r.indices)
            assert np.array_equal(b.average_distance, r.average_distance)


def test_knn_shifted_domain_golden():
    g = gold("knn")
    xs, ys, qx, qy = g["shift_x"], g["shift_y"], g["shift_qx"], g["shift_qy"]
    _, index = _grid_for(xs, ys, qx, qy, 2.0)
    r = A.knn_stage(A.PointSet(qx, qy), index, A.PointSet(xs, ys), 10)
    assert np.array_equal(r.distances_sq, g["shift_d2"])
    assert np.array_equal(r.average_distance, g["shift_avg"])


@pytest.mark.parametrize("k", [1, 3, 10, 15, 30, 64, 100])
def test_knn_random_vs_oracle(k):
    xs, ys, _ = O.generate_points(20_000, UNIT, 100 + k)
    qx, qy = O.generate_queries(3000, (-0.1, -0.1, 1.1, 1.1), 200 + k)
    cfg_o, index = _grid_for(xs, ys, qx, qy, 4.0)
    grid_o = O.build_index(xs, ys, cfg_o)
    d2, ids, avg, exh = O.knn_grid(qx, qy, cfg_o, grid_o, xs.size, k)
    r = A.knn_stage(A.PointSet(qx, qy), index, A.PointSet(xs, ys), k)
    assert np.array_equal(r.distances_sq, d2)
    assert np.array_equal(r.indices, ids)
    assert np.array_equal(r.average_distance, avg)


def test_knn_clustered_golden():
    g = gold("clustered")
    _, index = _grid_for(g["x"], g["y"], g["qx"], g["qy"], 4.0)
    r = A.knn_stage(A.PointSet(g["qx"], g["qy"]), index, A.PointSet(g["x"], g["y"]), 10)
    assert np.array_equal(r.distances_sq, g["d2"])
    assert np.array_equal(r.average_distance, g["avg"])


def test_knn_errors():  # test_knn.cpp:281-295
    xs, ys, _ = O.generate_points(800, UNIT, 31)
    qx, qy = O.generate_queries(120, UNIT, 32)
    _, index = _grid_for(xs, ys, qx, qy, 4.0)
    bad_x = qx.copy()
    bad_x[17] = 50.0
    with pytest.raises(A.AidwRuntimeError) as e:
        A.knn_stage(A.PointSet(bad_x, qy), index, A.PointSet(xs, ys), 5)
    assert "query 17" in str(e.value)
    with pytest.raises(A.InvalidArgument):
        A.knn_stage(A.PointSet(qx, qy), None, A.PointSet(xs, ys), 5, engine="grid")
    assert len(A.knn_stage(A.PointSet(), index, A.PointSet(xs, ys), 5)) == 0
    with pytest.raises(A.AidwRuntimeError):
        A.knn_stage(A.PointSet(qx, qy), None, A.PointSet(xs, ys), 801, engine="brute")


# ------------------------------------------------------------------ K3 + K4
def test_pipeline_10k_golden():
    """BASELINE configs[0]: 10K x 10K uniform, k = 10."""
    g = gold("pipeline10k")
    data = A.generate_random_points(10_000, UNIT, 42)
    queries = A.generate_random_queries(10_000, UNIT, 43)
    out = A.run_pipeline(data, queries, A.RunConfig(params=A.AidwParams(k=10)))
    alpha = out.result.alphas
    sat = g["alpha"] == 4.0
    assert np.array_equal(alpha[sat], g["alpha"][sat])
    assert rel_err(alpha, g["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, g["pred_blocked"], data.zs) <= FP32_TOL
    assert out.k_effective == 10
    A.set_weight_precision("fp64")  # blocked -> FP64 blocked-variant kernel
    out64 = A.run_pipeline(data, queries, A.RunConfig(params=A.AidwParams(k=10)))
    assert rel_err(out64.result.predicted, g["pred_blocked"]) <= FP64_TOL
    assert rel_err(out64.result.predicted, g["pred_naive"]) <= FP64_TOL
    naive = A.run_pipeline(data, queries, A.RunConfig(variant="naive", params=A.AidwParams(k=10)))
    assert rel_err(naive.result.predicted, g["pred_naive"]) <= FP64_TOL


def test_pipeline_clustered_golden():
    g = gold("clustered")
    data = A.PointSet(g["x"], g["y"], g["z"])
    out = A.run_pipeline(data, A.PointSet(g["qx"], g["qy"]), A.RunConfig(params=A.AidwParams(k=10)))
    assert rel_err(out.result.alphas, g["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, g["pred_blocked"], g["z"]) <= FP32_TOL


def test_predict_golden_idw_and_aidw():
    g = gold("predict")
    data = A.PointSet(g["idw_x"], g["idw_y"], g["idw_z"])
    q = A.PointSet(g["idw_qx"], g["idw_qy"])
    r = A.idw_predict_all(q, data, 2.0, "blocked")
    assert pred_err(r.predicted, g["idw_naive"], data.zs) <= FP32_TOL
    assert np.all(r.alphas == 2.0)
    n64 = A.idw_predict_all(q, data, 2.0, "naive")
    p64 = A.idw_predict_all(q, data, 2.0, "blocked", pinned_order=True)
    assert rel_err(n64.predicted, g["idw_naive"]) <= FP64_TOL
    assert np.array_equal(n64.predicted, p64.predicted)  # pinned == naive, bit-equal
    # AIDW radial, k = 15, queries past the hull
    data = A.PointSet(g["aidw_x"], g["aidw_y"], g["aidw_z"])
    q = A.PointSet(g["aidw_qx"], g["aidw_qy"])
    cfg = A.RunConfig(params=A.AidwParams(k=15))
    out = A.run_pipeline(data, q, cfg)
    assert rel_err(out.result.alphas, g["aidw_alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, g["aidw_blocked"], data.zs) <= FP32_TOL
    lo, hi = data.zs.min(), data.zs.max()
    assert np.all(out.result.predicted >= lo) and np.all(out.result.predicted <= hi)


def test_drop_in_chain_matches_pipeline():
    """build_index -> knn_stage -> aidw_predict_all equals the fused path."""
    data = A.generate_random_points(30_000, UNIT, 5, "planar")
    q = A.generate_random_queries(4000, UNIT, 6)
    bb = A.compute_bbox(data, q)
    index = A.build_index(data, A.make_grid_config(bb, A.choose_cell_width(data, bb, 4.0)))
    knn = A.knn_stage(q, index, data, 15)
    chained = A.aidw_predict_all(q, data, knn, A.AidwParams(k=15))
    fused = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=15)))
    assert np.array_equal(chained.alphas, fused.result.alphas)
    assert np.array_equal(chained.predicted, fused.result.predicted)


def test_constant_collapse_bit_equal():  # acceptance.cpp:215-234
    data = A.generate_random_points(1000, UNIT, 41)
    q = A.generate_random_queries(1000, UNIT, 42)
    params = A.AidwParams(alpha_levels=(2.0,) * 5)
    for variant in ("blocked", "naive"):
        bb = A.compute_bbox(data, q)
        index = A.build_index(data, A.make_grid_config(bb, A.choose_cell_width(data, bb, 4.0)))
        knn = A.knn_stage(q, index, data, params.k)
        adaptive = A.aidw_predict_all(q, data, knn, params, variant)
        constant = A.idw_predict_all(q, data, 2.0, variant)
        assert np.array_equal(adaptive.predicted, constant.predicted)
        assert np.all(adaptive.alphas == 2.0)


def test_snap_and_degenerate_fallback():
    data = A.generate_random_points(600, UNIT, 50, "radial")
    sites = A.PointSet(data.xs[:50], data.ys[:50])
    for variant in ("naive", "blocked"):
        r = A.idw_predict_all(sites, data, 2.0, variant)
        assert np.array_equal(r.predicted, data.zs[:50])
        a = A.run_pipeline(data, sites, A.RunConfig(variant=variant))
        assert np.array_equal(a.result.predicted, data.zs[:50])
    # test_interpolate.cpp:251-266: weights overflow -> nearest value
    d = A.PointSet([0.0, 1.0e-160], [0.0, 0.0], [3.0, 9.0])
    for variant in ("naive", "blocked"):
        r = A.idw_predict_all(A.PointSet([4.0e-161], [0.0]), d, 2.0, variant)
        assert r.predicted[0] == 3.0


def test_interpolation_properties_10k():  # acceptance.cpp:236-333 (FP32 tolerances)
    data = A.generate_random_points(10240, UNIT, 51, "planar")
    wide = A.generate_random_queries(200, (-0.2, -0.2, 1.2, 1.2), 52)
    base = A.run_pipeline(data, wide, A.RunConfig())
    lo, hi = data.zs.min(), data.zs.max()
    assert np.all(np.isfinite(base.result.predicted))
    assert np.all((base.result.predicted >= lo) & (base.result.predicted <= hi))
    moved = A.run_pipeline(A.PointSet(data.xs + 3.25, data.ys - 1.5, data.zs),
                           A.PointSet(wide.xs + 3.25, wide.ys - 1.5), A.RunConfig())
    diff = np.abs(moved.result.predicted - base.result.predicted)
    assert np.all(diff <= 1e-6 * np.maximum(1.0, np.abs(base.result.predicted)))
    A.set_weight_precision("fp64")
    b64 = A.run_pipeline(data, wide, A.RunConfig())
    m64 = A.run_pipeline(A.PointSet(data.xs + 3.25, data.ys - 1.5, data.zs),
                         A.PointSet(wide.xs + 3.25, wide.ys - 1.5), A.RunConfig())
    assert np.all(np.abs(m64.result.predicted - b64.result.predicted)
                  <= 1e-9 * np.maximum(1.0, np.abs(b64.result.predicted)))
    lat = [(x, y) for y in (0.2, 0.35, 0.5, 0.65, 0.8) for x in (0.2, 0.35, 0.5, 0.65, 0.8)]
    lq = A.PointSet([p[0] for p in lat], [p[1] for p in lat])
    r = A.run_pipeline(data, lq, A.RunConfig())
    truth = 1.5 * lq.xs - 2.5 * lq.ys + 4.0
    assert np.max(np.abs(r.result.predicted - truth) / np.abs(truth)) <= 0.05


def test_aidw_predict_all_errors():  # test_interpolate.cpp:237-281
    data = A.generate_random_points(100, UNIT, 95)
    q = A.PointSet([0.5], [0.5])
    bb = A.compute_bbox(data, q)
    index = A.build_index(data, A.make_grid_config(bb, A.choose_cell_width(data, bb, 4.0)))
    knn = A.knn_stage(q, index, data, 5)
    with pytest.raises(A.AidwRuntimeError) as e:
        A.aidw_predict_all(q, data, knn, A.AidwParams(k=7))
    assert "query 0" in str(e.value)
    with pytest.raises(A.InvalidArgument):
        A.aidw_predict_all(A.PointSet([0.5, 0.2], [0.5, 0.2]), data, knn, A.AidwParams(k=5))
    with pytest.raises(A.InvalidArgument):
        A.idw_predict_all(q, data, 0.0)
    with pytest.raises(A.InvalidArgument):
        A.idw_predict_all(q, A.PointSet([0.0], [0.0]), 2.0)


def test_brute_engine_pipeline_identical():  # acceptance.cpp:356-414 (outputs identical)
    data = A.generate_random_points(20_000, UNIT, 61)
    q = A.generate_random_queries(5000, UNIT, 62)
    g = A.run_pipeline(data, q, A.RunConfig())
    b = A.run_pipeline(data, q, A.RunConfig(knn_engine="brute"))
    assert np.array_equal(g.result.predicted, b.result.predicted)
    assert np.array_equal(g.result.alphas, b.result.alphas)


# ------------------------------------------------------------------ full size
def test_pipeline_1m_properties():
    """BASELINE configs[2] size: kNN bit-exact on a query sample, predictions
    within tolerance on a stratified sample, alpha distribution sane."""
    m = n = 1_000_000
    data = A.generate_random_points(m, UNIT, 42)
    q = A.generate_random_queries(n, UNIT, 43)
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    pred, alpha = out.result.predicted, out.result.alphas
    assert np.all(np.isfinite(pred))
    assert np.all((pred >= data.zs.min()) & (pred <= data.zs.max()))
    assert 0.9 < np.mean(alpha == 4.0) < 1.0
    assert out.stats["pairs"] == m * n
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(n, 128, replace=False))
    qs = A.PointSet(q.xs[sample], q.ys[sample])
    # kNN for the sample through the oracle's grid (same grid: bbox of all points)
    bb = O.compute_bbox(data.xs, data.ys, q.xs, q.ys)
    cfg_o = O.make_grid_config(bb, O.choose_cell_width(m, bb, 4.0))
    grid_o = O.build_index(data.xs, data.ys, cfg_o)
    d2, ids, avg, _ = O.knn_grid(qs.xs, qs.ys, cfg_o, grid_o, m, 10)
    rec = [O.adaptive_alpha(a, m, (bb[2] - bb[0]) * (bb[3] - bb[1]), k=10) for a in avg]
    ref_alpha = np.array([r[4] for r in rec])
    assert rel_err(alpha[sample], ref_alpha) <= 1e-12
    ref_pred = O.predict_with_alphas(qs.xs, qs.ys, data.xs, data.ys, data.zs, ref_alpha, 1)
    assert pred_err(pred[sample], ref_pred, data.zs) <= FP32_TOL
