"""GPU edge cases beyond the golden fixtures: exact distance ties and
duplicate points (index tie-break), lattice data, parameter quirks
(r_min != 0, explicit area, jumbled levels), idw mode, tiny / degenerate
sizes, shifted and scaled domains, error paths.  Oracle: the C restatement
(pinned to the reference in tests/test_oracle.py)."""
import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu
UNIT = (0.0, 0.0, 1.0, 1.0)


def pred_err(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * max(span, 1e-300))))


def grid_for(xs, ys, qx, qy, factor=4.0):
    bb = O.compute_bbox(xs, ys, qx, qy)
    cfg = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, factor))
    g = A.build_index(A.PointSet(xs, ys),
                      A.GridConfig(cfg.cell_width, cfg.n_col, cfg.n_row, cfg.min_x, cfg.min_y))
    return cfg, g


@pytest.fixture(autouse=True)
def fp32_default():
    A.set_weight_precision("fp32")
    yield
    A.set_weight_precision("fp32")


def test_lattice_ties_index_tiebreak():
    # integer lattice with duplicated points: many exactly equal distances
    gx, gy = np.meshgrid(np.arange(40.0), np.arange(30.0))
    xs = np.concatenate([gx.ravel(), gx.ravel()[::7]])
    ys = np.concatenate([gy.ravel(), gy.ravel()[::7]])
    qx = np.array([0.5, 10.0, 19.5, 39.0, 0.0, 20.25])
    qy = np.array([0.5, 10.0, 14.5, 29.0, 29.0, 14.75])
    cfg, g = grid_for(xs, ys, qx, qy)
    for k in (1, 4, 8, 13, 30):
        r = A.knn_stage(A.PointSet(qx, qy), g, A.PointSet(xs, ys), k)
        d2, ids, avg = O.knn_brute(qx, qy, xs, ys, k)
        assert np.array_equal(r.distances_sq, d2)
        assert np.array_equal(r.indices, ids)  # ties broken by index
        assert np.array_equal(r.average_distance, avg)


def test_all_points_identical():
    xs = np.full(50, 0.25)
    ys = np.full(50, 0.75)
    qx = np.array([0.25, 0.0, 1.0])
    qy = np.array([0.75, 0.0, 1.0])
    cfg, g = grid_for(np.append(xs, 0.9), np.append(ys, 0.1), qx, qy)
    xs2, ys2 = np.append(xs, 0.9), np.append(ys, 0.1)
    r = A.knn_stage(A.PointSet(qx, qy), g, A.PointSet(xs2, ys2), 10)
    d2, ids, _ = O.knn_brute(qx, qy, xs2, ys2, 10)
    assert np.array_equal(r.distances_sq, d2) and np.array_equal(r.indices, ids)
    zs = np.arange(51, dtype=float)
    out = A.run_pipeline(A.PointSet(xs2, ys2, zs), A.PointSet(qx, qy),
                         A.RunConfig(params=A.AidwParams(k=10)))
    assert out.result.predicted[0] == 0.0  # snaps to the FIRST coincident index


@pytest.mark.parametrize("params", [
    dict(k=7, r_min=0.5, r_max=2.0),                     # the pi / r_max quirk
    dict(k=12, r_min=0.0, r_max=1.5, area=2.0),           # explicit area
    dict(k=9, alpha_levels=(3.0, 0.5, 4.0, 1.0, 2.0)),    # jumbled levels
    dict(k=20, alpha_levels=(0.3, 0.7, 1.1, 2.9, 7.5)),   # non half-integer levels
])
def test_param_variants_vs_oracle(params):
    data = A.generate_random_points(6000, UNIT, 17, "radial")
    q = A.generate_random_queries(1500, (-0.05, -0.05, 1.05, 1.05), 18)
    p = A.AidwParams(**params)
    out = A.run_pipeline(data, q, A.RunConfig(params=p))
    ref = O.pipeline(data.xs, data.ys, data.zs, q.xs, q.ys, k=p.k, variant=0, r_min=p.r_min,
                     r_max=p.r_max, levels=p.alpha_levels, area=p.area)
    a_err = np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"])
    assert a_err <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], data.zs) <= 1e-5
    A.set_weight_precision("fp64")
    out64 = A.run_pipeline(data, q, A.RunConfig(params=p))
    assert np.max(np.abs(out64.result.predicted - ref["pred"]) / np.abs(ref["pred"])) <= 2e-11


@pytest.mark.parametrize("alpha", [0.5, 1.0, 1.7, 2.0, 3.0, 4.0, 8.0])
def test_idw_mode_vs_oracle(alpha):
    data = A.generate_random_points(20_000, UNIT, 3, "planar")
    q = A.generate_random_queries(700, UNIT, 4)
    out = A.run_pipeline(data, q, A.RunConfig(mode="idw", alpha=alpha))
    ref = O.predict_with_alphas(q.xs, q.ys, data.xs, data.ys, data.zs, np.full(q.count(), alpha), 0)
    assert pred_err(out.result.predicted, ref, data.zs) <= 1e-5
    assert np.all(out.result.alphas == alpha) and out.k_effective == 0


@pytest.mark.parametrize("scale", [1.0, 1e-3])
@pytest.mark.parametrize("levels,exact", [((2.0, 2.0, 3.0, 4.0, 4.0), (2.0, 4.0)),
                                          ((1.0, 1.0, 3.0, 3.0, 4.0), (1.0, 3.0, 4.0)),
                                          ((1.0, 1.0, 2.0, 2.0, 3.0), (1.0, 2.0, 3.0))])
def test_mixed_recipe_classes(scale, levels, exact):
    # levels saturating at exact integers on clustered data: warps mix the
    # recipe classes (alpha = 1, 2, 3, 4) with each other and with
    # general-alpha queries; a small domain exercises the per-query ratio
    # scaling (s != 1) of alpha 4
    xs, ys, zs = O.generate_clustered(30_000, seed=11)
    xs, ys = xs * scale, ys * scale
    qx, qy = O.generate_queries(3000, (0.0, 0.0, scale, scale), 12)
    p = A.AidwParams(k=10, alpha_levels=levels)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy), A.RunConfig(params=p))
    ref = O.pipeline(xs, ys, zs, qx, qy, k=10, variant=1, levels=p.alpha_levels)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    for a in exact:
        assert np.any(out.result.alphas == a)
    assert pred_err(out.result.predicted, ref["pred"], zs) <= 1e-5


def test_tiny_sizes():
    # m = 1: every prediction is the single value
    one = A.PointSet([0.3], [0.4], [42.0])
    q = A.PointSet([0.9, 0.3], [0.9, 0.4])
    assert A.idw_predict_all(q, one, 2.0).predicted.tolist() == [42.0, 42.0]
    # k clamps to m in run_pipeline (cli.hpp:237-238)
    data = A.generate_random_points(5, UNIT, 2)
    qq = A.generate_random_queries(9, UNIT, 3)
    out = A.run_pipeline(data, qq, A.RunConfig(params=A.AidwParams(k=15)))
    assert out.k_effective == 5
    ref = O.pipeline(data.xs, data.ys, data.zs, qq.xs, qq.ys, k=5, variant=1)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], data.zs) <= 1e-5
    # empty query set
    assert A.run_pipeline(data, A.PointSet(), A.RunConfig()).result.predicted.size == 0


@pytest.mark.parametrize("box", [(-3.0, 5.0, 17.0, 25.0), (1e6, -2e6, 1e6 + 3.0, -2e6 + 1.0),
                                 (0.0, 0.0, 1e-9, 1e-9), (-1e150, -1e150, 1e150, 1e150)])
def test_scaled_and_shifted_domains(box):
    data = A.generate_random_points(8000, box, 23, "radial")
    q = A.generate_random_queries(600, box, 24)
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    ref = O.pipeline(data.xs, data.ys, data.zs, q.xs, q.ys, k=10, variant=0)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], data.zs) <= 1e-5


def test_values_spanning_zero_and_large_magnitudes():
    data = A.generate_random_points(10_000, UNIT, 5)
    for zs in (data.zs * 2e30 - 1e30, (data.zs - 0.5) * 1e-30, data.zs + 1e6):
        d = A.PointSet(data.xs, data.ys, zs)
        q = A.generate_random_queries(500, UNIT, 6)
        out = A.run_pipeline(d, q, A.RunConfig(params=A.AidwParams(k=10)))
        ref = O.pipeline(d.xs, d.ys, d.zs, q.xs, q.ys, k=10, variant=0)
        assert pred_err(out.result.predicted, ref["pred"], zs) <= 1e-5


def test_error_paths():
    data = A.generate_random_points(100, UNIT, 1)
    with pytest.raises(A.InvalidArgument):
        A.run_pipeline(data, A.PointSet([0.5], [0.5]), A.RunConfig(params=A.AidwParams(r_min=2.0)))
    with pytest.raises(A.InvalidArgument):
        A.run_pipeline(A.PointSet([0.1, 0.2], [0.1, 0.2]), A.PointSet([0.1], [0.1]),
                       A.RunConfig())  # no values
    with pytest.raises(A.InvalidArgument):
        A.run_pipeline(data, A.PointSet([0.5], [0.5]), A.RunConfig(workers=-1))
    cfg, g = grid_for(data.xs, data.ys, np.array([0.5]), np.array([0.5]))
    with pytest.raises(A.AidwRuntimeError) as e:
        A.knn_stage(A.PointSet([0.5, float("nan")], [0.5, 0.5]), g, data, 3)
    assert "query 1" in str(e.value)
    knn = A.knn_stage(A.PointSet([0.5], [0.5]), g, data, 3)
    knn.average_distance[:] = float("nan")
    with pytest.raises(A.AidwRuntimeError) as e:
        A.aidw_predict_all(A.PointSet([0.5], [0.5]), data, knn, A.AidwParams(k=3))
    assert "alpha_from_mu" in str(e.value)
    knn.average_distance[:] = -1.0
    with pytest.raises(A.AidwRuntimeError) as e:
        A.aidw_predict_all(A.PointSet([0.5], [0.5]), data, knn, A.AidwParams(k=3))
    assert "rObs" in str(e.value)


def test_deterministic_and_shard_invariant():
    """Same query evaluated alone, in a shard, or in the full set gives the
    same bits (the multi-GPU invariance argument), given the global bbox."""
    data = A.generate_random_points(50_000, UNIT, 8)
    q = A.generate_random_queries(6000, UNIT, 9)
    bb = O.compute_bbox(data.xs, data.ys, q.xs, q.ys)
    cfg = A.RunConfig(params=A.AidwParams(k=10), bbox=tuple(bb))
    full = A.run_pipeline(data, q, cfg).result
    for lo, hi in ((0, 3000), (3000, 6000), (1234, 1240)):
        part = A.run_pipeline(data, A.PointSet(q.xs[lo:hi], q.ys[lo:hi]), cfg).result
        assert np.array_equal(part.predicted, full.predicted[lo:hi])
        assert np.array_equal(part.alphas, full.alphas[lo:hi])
    again = A.run_pipeline(data, q, cfg).result
    assert np.array_equal(again.predicted, full.predicted)


def test_workspace_reuse_across_sizes_and_threads():
    """The per-call device workspace (bump-allocated temporaries, recycled
    after each call, grown after an overflowing call): small -> large ->
    small calls, and calls from concurrent host threads, reproduce the bits
    of the first evaluation."""
    import threading
    small_d, small_q = A.generate_random_points(20_000, UNIT, 21), A.generate_random_queries(3000, UNIT, 22)
    big_d, big_q = A.generate_random_points(300_000, UNIT, 23), A.generate_random_queries(40_000, UNIT, 24)
    cfg = A.RunConfig(params=A.AidwParams(k=10))
    ref_small = A.run_pipeline(small_d, small_q, cfg).result.predicted
    ref_big = A.run_pipeline(big_d, big_q, cfg).result.predicted  # overflows, grows
    assert np.array_equal(A.run_pipeline(small_d, small_q, cfg).result.predicted, ref_small)
    assert np.array_equal(A.run_pipeline(big_d, big_q, cfg).result.predicted, ref_big)
    out = {}

    def work(i):
        d, q, ref = (small_d, small_q, ref_small) if i % 2 else (big_d, big_q, ref_big)
        out[i] = np.array_equal(A.run_pipeline(d, q, cfg).result.predicted, ref)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert all(out.values()) and len(out) == 4


@pytest.mark.parametrize("m", [2, 255, 256, 257, 2047, 2048, 2049, 4097, 262_144, 262_145])
def test_tile_and_chunk_boundaries(m):
    """Data sizes at the K4 tile (256), chunk-split (one tile per chunk up to
    64 chunks, 64 chunks up to 1024 tiles, 32 beyond) and nearest-search grid (4096)
    boundaries: partial last tiles are NEAR with exact-zero pads, every
    chunk is folded once — predictions within the contract, alpha exact."""
    data = A.generate_random_points(m, UNIT, 31)
    q = A.generate_random_queries(257, UNIT, 32)
    k = min(10, m)
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    ref = O.pipeline(data.xs, data.ys, data.zs, q.xs, q.ys, k=k, variant=1)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], data.zs) <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_query_slabs_bit_identical(precision):
    """The weighting runs its queries in slabs (aidw_set_query_slab) so its
    FP64 partial sums are bounded for any n: 3 / 1 KiB-query slabs give the
    bits of one slab, for AIDW (both query classes, general and alpha = 4
    regions straddling slab boundaries) and constant-alpha IDW."""
    data = A.generate_clustered(60_000, seed=3)
    q = A.generate_random_queries(10_000, UNIT, 4)
    A.set_weight_precision(precision)
    cfg = A.RunConfig(params=A.AidwParams(k=10))
    icfg = A.RunConfig(mode="idw", alpha=2.5)
    try:
        A.set_query_slab(0)
        ref = A.run_pipeline(data, q, cfg).result
        ref_idw = A.run_pipeline(data, q, icfg).result
        for slab in (3072, 1024):
            A.set_query_slab(slab)
            got = A.run_pipeline(data, q, cfg).result
            assert np.array_equal(got.predicted, ref.predicted)
            assert np.array_equal(got.alphas, ref.alphas)
            assert np.array_equal(A.run_pipeline(data, q, icfg).result.predicted, ref_idw.predicted)
    finally:
        A.set_query_slab(0)
    assert 0.05 < np.mean(ref.alphas == 4.0) < 0.95  # both K4 regions populated


def test_empty_queries_and_zero_area():
    """run_pipeline with n = 0 returns empty results (brute engine too);
    a zero-area bbox fails in the grid engine's cell width
    (choose_cell_width, invalid_argument) as in the reference (cli.hpp:240-248)."""
    data = A.generate_random_points(500, UNIT, 5)
    for engine in ("grid", "brute"):
        out = A.run_pipeline(data, A.PointSet(), A.RunConfig(knn_engine=engine))
        assert out.result.predicted.size == 0
    line = A.PointSet(np.linspace(0, 1, 50), np.full(50, 0.5), np.arange(50.0))
    with pytest.raises(A.InvalidArgument) as e:
        A.run_pipeline(line, A.PointSet([0.5], [0.5]), A.RunConfig())
    assert "choose_cell_width" in str(e.value)
    with pytest.raises(A.InvalidArgument):
        A.run_pipeline(line, A.PointSet(), A.RunConfig())


@pytest.mark.parametrize("mode", ["aidw", "idw"])
def test_graph_replay_bit_identical(mode):
    """A repeated pass (same plan, buffers, workspace) is captured into a
    CUDA graph and replayed: the replays give the eager pass's bits, count
    their kernels, and time their stages."""
    data = A.generate_random_points(30_000, UNIT, 12)
    q = A.generate_random_queries(7_000, UNIT, 13)
    cfg = A.RunConfig(mode=mode, params=A.AidwParams(k=10), alpha=3.0)
    A.set_graphs(False)
    try:
        ref = A.run_pipeline(data, q, cfg)
    finally:
        A.set_graphs(True)
    c0 = A.graph_counters()
    outs = [A.run_pipeline(data, q, cfg) for _ in range(5)]
    c1 = A.graph_counters()
    assert c1["captures"] >= c0["captures"] + 1 and c1["replays"] >= c0["replays"] + 2
    for o in outs:
        assert np.array_equal(o.result.predicted, ref.result.predicted)
        assert np.array_equal(o.result.alphas, ref.result.alphas)
    last = outs[-1].stats
    assert last["kernel_launches"] == ref.stats["kernel_launches"]
    assert last["weight_kernel_ms"] > 0 and last["interp_ms"] > 0
    assert last["alpha4_queries"] == ref.stats["alpha4_queries"]
