"""Pin the C restatement (oracle/aidw_oracle.c) before trusting it.

Two anchors (CPU only, no GPU needed):
  1. the reference's own known-answer tests (proj/tests/test_*.cpp frozen
     values), restated here against the oracle;
  2. the golden fixtures in tests/golden/, produced by the reference itself
     (tests/golden/make_golden.py), compared bit-for-bit where the reference
     is bit-reproducible and within the reference's own tolerances otherwise.
When oracle/_ref/libaidw_ref.so is present the oracle is also cross-checked
against the live reference on fresh random instances.
"""
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
UNIT = (0.0, 0.0, 1.0, 1.0)
LEVELS = (0.5, 1.0, 2.0, 3.0, 4.0)


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


# ------------------------------------------------------------ known answers
def test_dist_sq_frozen():  # test_knn.cpp:40-44
    assert O.dist_sq(0.0, 0.0, 3.0, 4.0) == 25.0
    assert O.dist_sq(1.0, 1.0, 1.0, 1.0) == 0.0
    assert O.dist_sq(-1.0, -2.0, 2.0, 2.0) == 25.0


def test_brute_frozen():  # test_knn.cpp:46-66
    d2, ids, avg = O.knn_brute([2.0], [3.0], [2.0, 5.0], [3.0, 5.0], 1)
    assert d2[0].tolist() == [0.0] and avg[0] == 0.0
    d2, ids, avg = O.knn_brute([0.0], [0.0], [0.0, 3.0, 0.0], [0.0, 0.0, 4.0], 2)
    assert d2[0].tolist() == [0.0, 9.0] and avg[0] == 1.5
    assert ids[0].tolist() == [0, 1]


def test_brute_rejects_bad_k():  # test_knn.cpp:87-93
    xs, ys, _ = O.generate_points(10, UNIT, 1)
    with pytest.raises(O.OracleError):
        O.knn_brute([0.5], [0.5], xs, ys, 0)
    with pytest.raises(O.OracleError):
        O.knn_brute([0.5], [0.5], xs, ys, 11)


def test_grid_geometry_frozen():  # test_grid.cpp:26-38, :67-83, :85-112
    box = (0.0, 0.0, 10.0, 10.0)
    assert O.choose_cell_width(100, box, 1.0) == 0.5
    assert O.choose_cell_width(400, box, 1.0) == 0.25
    assert O.choose_cell_width(400, box, 4.0) == 1.0
    cfg = O.make_grid_config((0.0, 0.0, 10.0, 4.0), 1.0)
    assert (cfg.n_col, cfg.n_row) == (11, 5)
    with pytest.raises(O.OracleError):
        O.make_grid_config((0.0, 0.0, 1.0, 1.0), 1.0e-9)
    c6 = O.grid_config(1.0, 6, 6)
    assert O.locate_cell(2.5, 3.5, c6) == (2, 3)
    assert O.locate_cell(-1.0e-12, 0.0, c6) == (0, 0)
    assert O.locate_cell(6.0, 6.0, c6) == (5, 5)
    with pytest.raises(O.OracleError) as e:
        O.locate_cell(-1.0, 0.0, c6)
    assert e.value.code == 2  # domain_error


def test_build_index_2x2():  # test_grid.cpp:150-170
    cfg = O.grid_config(1.0, 2, 2)
    ids, cs, sx, sy = O.build_index([1.5, 0.5, 1.5, 0.5], [0.5, 1.5, 1.5, 0.5], cfg)
    assert ids.tolist() == [3, 0, 1, 2]
    assert cs.tolist() == [0, 1, 2, 3, 4]


def test_fig4_regression():  # test_knn.cpp:167-200 / acceptance.cpp:123-161
    xs = [2.95, 2.95, 2.95, 1.98, 0.5, 4.5, 0.5, 4.5]
    ys = [2.50, 2.60, 2.40, 2.50, 0.5, 4.5, 4.5, 0.5]
    cfg = O.grid_config(1.0, 5, 5)
    grid = O.build_index(xs, ys, cfg)
    d2, ids, avg, exh = O.knn_grid([2.05], [2.5], cfg, grid, 8, 3)
    assert d2[0, 0] == O.dist_sq(2.05, 2.5, 1.98, 2.5)
    assert ids[0, 0] == 3
    bd2, _, _ = O.knn_brute([2.05], [2.5], xs, ys, 3)
    assert np.array_equal(d2, bd2)


def test_exhaustion():  # test_knn.cpp:238-247
    xs, ys, _ = O.generate_points(5, UNIT, 2)
    cfg = O.make_grid_config(np.array(UNIT), 0.25)
    grid = O.build_index(xs, ys, cfg)
    d2, ids, avg, exh = O.knn_grid([0.5], [0.5], cfg, grid, 5, 64)
    assert exh[0]
    assert np.isinf(d2[0, 5:]).all()
    full = np.sort([O.dist_sq(0.5, 0.5, x, y) for x, y in zip(xs, ys)])
    assert np.array_equal(d2[0, :5], full)


def test_adaptive_frozen():  # test_adaptive.cpp:54-163
    assert O.adaptive_alpha(0.0, 100, 100.0, k=4)[0] == 0.5
    assert O.normalize_mu(0.0) == 0.0 and O.normalize_mu(2.0) == 1.0
    assert abs(O.normalize_mu(1.0) - 0.5) <= 1e-15
    for i, b in enumerate((0.1, 0.3, 0.5, 0.7, 0.9)):
        assert O.alpha_from_mu(b, LEVELS) == LEVELS[i]
    assert O.alpha_from_mu(0.2, LEVELS) == 0.5 * 0.5 + 0.5 * 1.0
    for mu in np.linspace(0, 1, 1001):
        assert O.alpha_from_mu(mu, (2.0,) * 5) == 2.0
    with pytest.raises(O.OracleError) as e:
        O.alpha_from_mu(float("nan"), LEVELS)
    assert e.value.code == 2
    below = O.normalize_mu(2.0 - 1e-12, 0.5, 2.0)
    assert below == 0.5 - 0.5 * math.cos(math.pi / 2.0 * (2.0 - 1e-12 - 0.5))
    rec = O.adaptive_alpha(0.5, 100, 100.0, k=4)
    assert rec[2] == 1.0 and abs(rec[4] - 2.0) <= 1e-12
    with pytest.raises(O.OracleError):
        O.adaptive_alpha(0.5, 100, 100.0, k=4, list_len=3)
    O.adaptive_alpha(0.5, 100, 100.0, k=4, list_len=3, exhausted=True)


def test_weighting_frozen():  # test_interpolate.cpp:33-86, :251-266
    p = O.predict_with_alphas([1.0], [1.0], [1.0, 2.0], [1.0, 2.0], [7.0, 3.0], [2.0])
    assert p[0] == 7.0
    for a in (0.5, 1.0, 2.0, 7.0):
        assert O.predict_with_alphas([1.0], [0.0], [0.0, 2.0], [0.0, 0.0], [0.0, 10.0], [a])[0] == 5.0
    p = O.predict_with_alphas([0.5], [0.0], [0.0, 2.0], [0.0, 0.0], [0.0, 4.0], [2.0])
    assert abs(p[0] - 0.4) <= 1e-14 * 0.4
    p = O.predict_with_alphas([0.1], [0.05], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 5.0, 9.0], [64.0])
    assert abs(p[0] - 1.0) <= 1e-3
    for v in (0, 1):
        p = O.predict_with_alphas([4.0e-161], [0.0], [0.0, 1.0e-160], [0.0, 0.0], [3.0, 9.0], [2.0], v)
        assert p[0] == 3.0


# ------------------------------------------------------------ golden fixtures
def test_golden_generate():
    g = gold("generate")
    for i in range(5):
        cnt, x0, y0, x1, y1, seed, rule = g[f"p{i}_args"]
        xs, ys, zs = O.generate_points(int(cnt), (x0, y0, x1, y1), int(seed), int(rule))
        assert np.array_equal(xs, g[f"p{i}_x"]) and np.array_equal(ys, g[f"p{i}_y"])
        assert np.array_equal(zs, g[f"p{i}_z"])
    cnt, x0, y0, x1, y1, seed = g["q_args"]
    qx, qy = O.generate_queries(int(cnt), (x0, y0, x1, y1), int(seed))
    assert np.array_equal(qx, g["q_x"]) and np.array_equal(qy, g["q_y"])


def test_golden_grid():
    g = gold("grid")
    for tag in ("a", "b"):
        c = g[f"{tag}_cfg"]
        cfg = O.grid_config(c[0], int(c[1]), int(c[2]), c[3], c[4])
        if tag == "a":
            bb = O.compute_bbox(g["a_x"], g["a_y"])
            mine = O.make_grid_config(bb, O.choose_cell_width(g["a_x"].size, bb, 4.0))
            assert (mine.cell_width, mine.n_col, mine.n_row) == (c[0], int(c[1]), int(c[2]))
        ids, cs, sx, sy = O.build_index(g[f"{tag}_x"], g[f"{tag}_y"], cfg)
        assert np.array_equal(ids, g[f"{tag}_ids"])
        assert np.array_equal(cs, g[f"{tag}_cell_start"])
        assert np.array_equal(sx, g[f"{tag}_sx"]) and np.array_equal(sy, g[f"{tag}_sy"])


@pytest.mark.parametrize("tag", ["std", "tiny", "exh"])
def test_golden_knn(tag):
    g = gold("knn")
    xs, ys, qx, qy = g[f"{tag}_x"], g[f"{tag}_y"], g[f"{tag}_qx"], g[f"{tag}_qy"]
    factor = float(g[f"{tag}_factor"][0])
    bb = O.compute_bbox(xs, ys, qx, qy)
    cfg = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, factor))
    grid = O.build_index(xs, ys, cfg)
    for k in g[f"{tag}_ks"]:
        k = int(k)
        d2, ids, avg, exh = O.knn_grid(qx, qy, cfg, grid, xs.size, k)
        assert np.array_equal(d2, g[f"{tag}_k{k}_d2"])
        assert np.array_equal(avg, g[f"{tag}_k{k}_avg"])
        assert np.array_equal(exh, g[f"{tag}_k{k}_exh"])
        if k <= xs.size:  # index sets: lexicographic (d2, idx) = brute force
            bd2, bids, bavg = O.knn_brute(qx, qy, xs, ys, k)
            assert np.array_equal(ids, bids) and np.array_equal(d2, bd2)


def test_golden_knn_shifted():
    g = gold("knn")
    xs, ys, qx, qy = g["shift_x"], g["shift_y"], g["shift_qx"], g["shift_qy"]
    bb = O.compute_bbox(xs, ys, qx, qy)
    cfg = O.make_grid_config(bb, O.choose_cell_width(xs.size, bb, 2.0))
    d2, ids, avg, _ = O.knn_grid(qx, qy, cfg, O.build_index(xs, ys, cfg), xs.size, 10)
    assert np.array_equal(d2, g["shift_d2"]) and np.array_equal(avg, g["shift_avg"])


def test_golden_adaptive():
    g = gold("adaptive")
    for j, (r, m, a) in enumerate(zip(g["r_obs"], g["m"], g["area"])):
        rec = O.adaptive_alpha(r, int(m), a, k=4, levels=LEVELS)
        assert np.array_equal(rec, g["rec"][j])  # same libm: bit-exact
        recj = O.adaptive_alpha(r, int(m), a, k=4, levels=tuple(g["jumbled"]), r_min=0.5)
        assert np.array_equal(recj, g["rec_jumbled"][j])


def test_golden_predict():
    g = gold("predict")
    qx, qy, xs, ys, zs = g["idw_qx"], g["idw_qy"], g["idw_x"], g["idw_y"], g["idw_z"]
    naive = O.predict_with_alphas(qx, qy, xs, ys, zs, np.full(qx.size, 2.0), 0)
    assert np.array_equal(naive, g["idw_naive"])          # naive: bit-exact
    assert np.array_equal(g["idw_pinned"], g["idw_naive"])  # reference pinned == naive
    blocked = O.predict_with_alphas(qx, qy, xs, ys, zs, np.full(qx.size, 2.0), 1)
    assert np.allclose(blocked, g["idw_blocked"], rtol=1e-12, atol=0)
    # AIDW: alphas bit-exact, naive predictions bit-exact
    xs, ys, zs, qx, qy = g["aidw_x"], g["aidw_y"], g["aidw_z"], g["aidw_qx"], g["aidw_qy"]
    out = O.pipeline(xs, ys, zs, qx, qy, k=15, variant=0)
    assert np.array_equal(out["alpha"], g["aidw_alpha"])
    assert np.array_equal(out["pred"], g["aidw_naive"])
    assert g["degen_naive"][0] == 3.0 and g["degen_blocked"][0] == 3.0


def test_golden_pipeline_10k():
    g = gold("pipeline10k")
    xs, ys, zs = O.generate_points(10000, UNIT, 42, 0)
    qx, qy = O.generate_queries(10000, UNIT, 43)
    out = O.pipeline(xs, ys, zs, qx, qy, k=10, variant=0)
    assert np.array_equal(out["d2"], g["d2"]) and np.array_equal(out["avg"], g["avg"])
    assert np.array_equal(out["alpha"], g["alpha"])
    assert np.array_equal(out["pred"], g["pred_naive"])
    rel = np.abs(out["pred"] - g["pred_blocked"]) / np.abs(g["pred_blocked"])
    assert rel.max() < 1e-12


def test_golden_clustered():
    g = gold("clustered")
    cx, cy, cz = O.generate_clustered(20000, seed=42)
    assert np.array_equal(cx, g["x"]) and np.array_equal(cz, g["z"])
    qx, qy = O.generate_clustered(5000, seed=43, with_values=False)
    out = O.pipeline(cx, cy, cz, qx, qy, k=10, variant=1)
    assert np.array_equal(out["d2"], g["d2"]) and np.array_equal(out["alpha"], g["alpha"])
    rel = np.abs(out["pred"] - g["pred_blocked"]) / np.abs(g["pred_blocked"])
    assert rel.max() < 1e-12


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_live_reference_random_instances():
    rng = np.random.default_rng(7)
    for inst in range(12):
        m = int(rng.integers(10, 3000)); n = int(rng.integers(1, 200))
        k = int(rng.choice([1, 3, 10, 30, 64]))
        factor = float(rng.choice([1.0, 2.0, 4.0, 8.0]))
        box = (-3.0, 5.0, 17.0, 25.0) if inst % 3 == 0 else UNIT
        xs, ys, zs = O.generate_points(m, box, 1000 + inst)
        qx, qy = O.generate_queries(n, box, 900000 + inst)
        rd2, ravg, rexh, _ = O.ref_knn_stage(qx, qy, xs, ys, k, engine=0, factor=factor)
        bb = O.compute_bbox(xs, ys, qx, qy)
        cfg = O.make_grid_config(bb, O.choose_cell_width(m, bb, factor))
        d2, ids, avg, exh = O.knn_grid(qx, qy, cfg, O.build_index(xs, ys, cfg), m, k)
        assert np.array_equal(d2, rd2) and np.array_equal(avg, ravg)
        assert np.array_equal(exh, rexh)
