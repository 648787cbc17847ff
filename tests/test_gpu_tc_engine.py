"""The tensor-core K4 engine (csrc/weight_tc.cu, selected when a data chunk
has >= 4 tiles, i.e. m >= 64K) on every query class it evaluates: the
recipe classes alpha = 4 / 2 / 1 / 3 (interpolate.hpp:174-209), warps that
mix them (kClsMixed), the per-query range scale of alpha = 4 on small
domains, partial last tiles and the near / far split — predictions within
the FP32 contract of the C oracle (pinned to the reference in
tests/test_oracle.py), alphas exact.  The CUDA-core engine covers the same
forms at m < 64K in test_gpu_edge.py / test_gpu_vs_reference.py."""
import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu
UNIT = (0.0, 0.0, 1.0, 1.0)
M = 80_000  # 313 tiles -> 64 chunks of 4-5 tiles: the tensor-core engine


def pred_err(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * max(span, 1e-300))))


@pytest.fixture(autouse=True)
def fp32_default():
    A.set_weight_precision("fp32")
    yield
    A.set_weight_precision("fp32")


def test_engine_selection():
    assert A.weight_engine(M) == "tensor-core"
    assert A.weight_engine(30_000) == "cuda-core"


@pytest.mark.parametrize("alpha", [1.0, 2.0, 3.0, 4.0])
def test_idw_recipe_classes(alpha):
    """Constant-alpha IDW: every query in one recipe class."""
    data = A.generate_random_points(M + 77, UNIT, 5, "planar")  # partial last tile
    q = A.generate_random_queries(1500, UNIT, 6)
    out = A.run_pipeline(data, q, A.RunConfig(mode="idw", alpha=alpha))
    ref = O.predict_with_alphas(q.xs, q.ys, data.xs, data.ys, data.zs,
                                np.full(q.count(), alpha), 0)
    assert pred_err(out.result.predicted, ref, data.zs) <= 1e-5


@pytest.mark.parametrize("scale", [1.0, 1e-3])
@pytest.mark.parametrize("levels,exact", [((2.0, 2.0, 3.0, 4.0, 4.0), (2.0, 4.0)),
                                          ((1.0, 1.0, 3.0, 3.0, 4.0), (1.0, 3.0, 4.0)),
                                          ((1.0, 1.0, 2.0, 2.0, 3.0), (1.0, 2.0, 3.0))])
def test_mixed_recipe_classes(scale, levels, exact):
    """Levels saturating at integers on clustered data: the recipe region
    holds several classes, warps straddling a class boundary run the mixed
    form, and the general-alpha queries go to the CUDA-core launch beside
    it; a 1e-3 domain exercises the alpha = 4 range scale s != 1."""
    xs, ys, zs = O.generate_clustered(M, seed=21)
    xs, ys = xs * scale, ys * scale
    qx, qy = O.generate_queries(2000, (0.0, 0.0, scale, scale), 22)
    p = A.AidwParams(k=10, alpha_levels=levels)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy), A.RunConfig(params=p))
    ref = O.pipeline(xs, ys, zs, qx, qy, k=10, variant=1, levels=p.alpha_levels)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    for a in exact:
        assert np.any(out.result.alphas == a)
    assert pred_err(out.result.predicted, ref["pred"], zs) <= 1e-5


def test_near_tiles_and_snaps():
    """Queries on and next to data sites (near tiles, snap tolerance) and
    duplicated sites: the hi/lo near form, exact snaps."""
    data = A.generate_random_points(M, UNIT, 7)
    rng = np.random.default_rng(8)
    pick = rng.choice(M, 800, replace=False)
    qx = np.concatenate([data.xs[pick], data.xs[pick[:400]] + 1e-6, rng.random(800)])
    qy = np.concatenate([data.ys[pick], data.ys[pick[:400]] - 1e-6, rng.random(800)])
    out = A.run_pipeline(data, A.PointSet(qx, qy), A.RunConfig(params=A.AidwParams(k=10)))
    ref = O.pipeline(data.xs, data.ys, data.zs, qx, qy, k=10, variant=1)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], data.zs) <= 1e-5
    assert np.array_equal(out.result.predicted[:800], data.zs[pick])  # snapped: exact values


def test_values_spanning_zero_and_large_magnitudes():
    """Zero-mean white-noise values of magnitude 1e30.  FP32 weights carry a
    few ulp each, so a prediction's absolute error is ~2e-7 of the value span
    whatever its size (tools/zero_cross_study.py: 1.9e-7 at 80K, both
    engines): the relative contract holds where |ref| >= 2 % of the span,
    the absolute one (1e-6 of the span) everywhere; FP64 mode is exact to
    2e-11 relative."""
    data = A.generate_random_points(M, UNIT, 9)
    zs = (data.zs - 0.5) * 1e30
    q = A.generate_random_queries(1000, UNIT, 10)
    d = A.PointSet(data.xs, data.ys, zs)
    out = A.run_pipeline(d, q, A.RunConfig(params=A.AidwParams(k=10)))
    ref = O.pipeline(data.xs, data.ys, zs, q.xs, q.ys, k=10, variant=1)
    span = float(zs.max() - zs.min())
    err = np.abs(out.result.predicted - ref["pred"])
    assert err.max() <= 1e-6 * span
    assert np.max(err / np.maximum(np.abs(ref["pred"]), 2e-2 * span)) <= 1e-5
    A.set_weight_precision("fp64")
    out64 = A.run_pipeline(d, q, A.RunConfig(params=A.AidwParams(k=10)))
    ref0 = O.pipeline(data.xs, data.ys, zs, q.xs, q.ys, k=10, variant=0)
    assert np.max(np.abs(out64.result.predicted - ref0["pred"]) / np.abs(ref0["pred"])) <= 2e-11


# ------------------------------------------------------------ invariances
def test_shard_invariant():
    """A query's bits do not depend on the other queries (its CTA, TMEM
    lane, warp-mates, class region): the multi-GPU argument, on the
    tensor-core engine."""
    data = A.generate_clustered(M, seed=31)
    q = A.generate_random_queries(6000, UNIT, 32)
    bb = O.compute_bbox(data.xs, data.ys, q.xs, q.ys)
    cfg = A.RunConfig(params=A.AidwParams(k=10), bbox=tuple(bb))
    full = A.run_pipeline(data, q, cfg).result
    assert 0.05 < np.mean(full.alphas == 4.0) < 0.95  # both K4 regions populated
    for lo, hi in ((0, 3000), (3000, 6000), (1234, 1240), (5999, 6000)):
        part = A.run_pipeline(data, A.PointSet(q.xs[lo:hi], q.ys[lo:hi]), cfg).result
        assert np.array_equal(part.predicted, full.predicted[lo:hi])
        assert np.array_equal(part.alphas, full.alphas[lo:hi])


def test_query_slabs_bit_identical():
    """Queries in slabs (bounded partial sums for any n): the slab bounds cut
    through the tensor-core recipe region and the general region."""
    data = A.generate_clustered(M, seed=33)
    q = A.generate_random_queries(10_000, UNIT, 34)
    cfg = A.RunConfig(params=A.AidwParams(k=10))
    try:
        A.set_query_slab(0)
        ref = A.run_pipeline(data, q, cfg).result
        for slab in (3072, 1000):
            A.set_query_slab(slab)
            got = A.run_pipeline(data, q, cfg).result
            assert np.array_equal(got.predicted, ref.predicted)
            assert np.array_equal(got.alphas, ref.alphas)
    finally:
        A.set_query_slab(0)


def test_graph_replay_bit_identical():
    data = A.generate_random_points(M, UNIT, 35)
    q = A.generate_random_queries(5_000, UNIT, 36)
    cfg = A.RunConfig(params=A.AidwParams(k=10))
    A.set_graphs(False)
    try:
        ref = A.run_pipeline(data, q, cfg).result
    finally:
        A.set_graphs(True)
    for _ in range(3):
        got = A.run_pipeline(data, q, cfg).result
        assert np.array_equal(got.predicted, ref.predicted)


def test_multidevice_shards_bit_identical():
    """Single-process multi-device path (query shards on three streams of
    device 0, data replicated by NCCL) on the tensor-core engine."""
    data = A.generate_random_points(M, UNIT, 37)
    q = A.generate_random_queries(20_001, UNIT, 38)
    cfg = A.RunConfig(params=A.AidwParams(k=10))
    one = A.run_pipeline(data, q, cfg).result
    A.set_devices([0, 0, 0])
    try:
        multi = A.run_pipeline(data, q, cfg).result
    finally:
        A.set_devices([])
    assert np.array_equal(multi.predicted, one.predicted)
    assert np.array_equal(multi.alphas, one.alphas)
