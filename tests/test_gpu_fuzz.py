"""Randomised differential testing of the fused pipeline against the C oracle
(pinned to the reference in tests/test_oracle.py): random sizes, k, cell
factors, engines, value rules, clustered / uniform / duplicated data,
shifted and scaled domains, alpha parameters.  Contract per case: alpha
bit-exact where mu saturates and <= 1e-12 otherwise, predictions within the
FP32 contract (FP64 mode: 2e-11)."""
import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu


def pred_err(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * max(span, 1e-300))))


def case(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.choice([3, 17, 256, 900, 4097, 12_000, 30_000]))
    n = int(rng.choice([1, 2, 31, 700, 3000]))
    x0, y0 = rng.uniform(-1e3, 1e3, 2)
    w = 10.0 ** rng.uniform(-3, 3)
    h = w * rng.uniform(0.2, 5.0)
    box = (x0, y0, x0 + w, y0 + h)
    kind = rng.choice(["uniform", "planar", "clustered", "dups"])
    if kind == "clustered":
        xs, ys, zs = O.generate_clustered(m, seed=seed)
        xs, ys = box[0] + xs * w, box[1] + ys * h
    else:
        xs, ys, zs = O.generate_points(m, box, seed, 1 if kind == "planar" else 0)
        if kind == "dups":
            k_d = max(1, m // 5)
            xs[:k_d] = xs[0]
            ys[:k_d] = ys[0]
    qx, qy = O.generate_queries(n, box, seed + 1)
    if rng.random() < 0.3:  # some queries exactly on data sites (snap)
        j = rng.integers(0, m, min(n, 5))
        qx[:j.size], qy[:j.size] = xs[j], ys[j]
    k = int(rng.choice([1, 3, 10, 15, 24, 70]))
    factor = float(rng.choice([1.0, 2.0, 4.0, 8.0]))
    r_max = float(rng.choice([1.5, 2.0, 3.0]))
    engine = str(rng.choice(["grid", "brute"]))
    return xs, ys, zs, qx, qy, k, factor, r_max, engine


@pytest.mark.parametrize("seed", range(200))
def test_pipeline_random_case(seed):
    xs, ys, zs, qx, qy, k, factor, r_max, engine = case(seed)
    data, q = A.PointSet(xs, ys, zs), A.PointSet(qx, qy)
    cfg = A.RunConfig(params=A.AidwParams(k=k, r_max=r_max), cell_factor=factor,
                      knn_engine=engine)
    out = A.run_pipeline(data, q, cfg)
    k_eff = min(k, xs.size)
    ref = O.pipeline(xs, ys, zs, qx, qy, k=k_eff, factor=factor, variant=1, r_max=r_max)
    assert out.k_effective == k_eff
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    assert pred_err(out.result.predicted, ref["pred"], zs) <= 1e-5


@pytest.mark.parametrize("seed", range(1000, 1040))
def test_pipeline_random_case_fp64(seed):
    xs, ys, zs, qx, qy, k, factor, r_max, engine = case(seed)
    A.set_weight_precision("fp64")
    try:
        out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                             A.RunConfig(params=A.AidwParams(k=k, r_max=r_max),
                                         cell_factor=factor, knn_engine=engine))
    finally:
        A.set_weight_precision("fp32")
    k_eff = min(k, xs.size)
    ref = O.pipeline(xs, ys, zs, qx, qy, k=k_eff, factor=factor, variant=1, r_max=r_max)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    span = float(np.max(zs) - np.min(zs))
    rel = np.abs(out.result.predicted - ref["pred"]) / np.maximum(np.abs(ref["pred"]),
                                                                  1e-3 * max(span, 1e-300))
    assert float(np.max(rel)) <= 2e-11


def case_tc(seed):
    """Sizes where K4 runs on the tensor-core engine (m >= 64K), with random
    levels (integer-saturating ones give the alpha = 1 / 2 / 3 recipe classes
    and mixed warps), domains, value rules and duplicated sites."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(65_600, 160_000))
    n = int(rng.choice([1, 33, 500, 1500]))
    x0, y0 = rng.uniform(-1e3, 1e3, 2)
    w = 10.0 ** rng.uniform(-3, 3)
    h = w * rng.uniform(0.3, 3.0)
    box = (x0, y0, x0 + w, y0 + h)
    kind = rng.choice(["uniform", "planar", "clustered", "dups"])
    if kind == "clustered":
        xs, ys, zs = O.generate_clustered(m, seed=seed)
        xs, ys = box[0] + xs * w, box[1] + ys * h
    else:
        xs, ys, zs = O.generate_points(m, box, seed, 1 if kind == "planar" else 0)
        if kind == "dups":
            k_d = max(1, m // 7)
            xs[:k_d] = xs[0]
            ys[:k_d] = ys[0]
    qx, qy = O.generate_queries(n, box, seed + 1)
    if rng.random() < 0.3:
        j = rng.integers(0, m, min(n, 5))
        qx[:j.size], qy[:j.size] = xs[j], ys[j]
    k = int(rng.choice([1, 5, 10, 15, 32]))
    levels = [(0.5, 1.0, 2.0, 3.0, 4.0), (1.0, 1.0, 2.0, 3.0, 4.0), (2.0, 2.0, 3.0, 4.0, 4.0),
              (1.0, 1.5, 2.5, 3.0, 3.0)][int(rng.integers(0, 4))]
    factor = float(rng.choice([2.0, 4.0, 8.0]))
    return xs, ys, zs, qx, qy, k, factor, levels


@pytest.mark.parametrize("seed", range(2000, 2060))
def test_pipeline_random_case_tensor_core_engine(seed):
    xs, ys, zs, qx, qy, k, factor, levels = case_tc(seed)
    assert A.weight_engine(xs.size) == "tensor-core"
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(params=A.AidwParams(k=k, alpha_levels=levels),
                                     cell_factor=factor))
    ref = O.pipeline(xs, ys, zs, qx, qy, k=k, factor=factor, variant=1, levels=levels)
    assert np.max(np.abs(out.result.alphas - ref["alpha"]) / ref["alpha"]) <= 1e-12
    span = float(zs.max() - zs.min())
    if zs.min() < 0.0 < zs.max():
        # a zero-crossing field (planar values on a shifted domain): FP32
        # weights leave an absolute error of ~1e-7 of the span, so the
        # relative contract applies where |ref| >= 2 % of the span
        # (DESIGN.md (c); seed 2048: 1.2e-8 of the span at |ref| = 0.3 %)
        err = np.abs(out.result.predicted - ref["pred"])
        assert err.max() <= 1e-6 * span
        assert np.max(err / np.maximum(np.abs(ref["pred"]), 2e-2 * span)) <= 1e-5
    else:
        assert pred_err(out.result.predicted, ref["pred"], zs) <= 1e-5
