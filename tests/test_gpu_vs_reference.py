"""The fused B200 pipeline against the reference's OWN cli::run_pipeline
(proj/include/aidw/cli.hpp:217-268, compiled in place into
oracle/_ref/libaidw_ref.so — test infrastructure only) on identical inputs:
uniform, clustered and planar data, AIDW with default and integer-saturating
levels, constant-alpha IDW on the recipe classes (alpha = 1, 2, 3, 4) and a
general alpha.  Contract (BASELINE north_star): alphas within 1e-12
relative (the FP64 chain is the reference's except the device cos in the
membership function: glibc and CUDA cos differ by an ulp), predictions
within 1e-5 * max(|ref|, 1e-3 * value span) in the default FP32 weighting
mode and 2e-11 in FP64 mode."""
import numpy as np
import pytest

import oracle as O
import paper_1601_05904_b200 as A

pytestmark = pytest.mark.gpu
UNIT = (0.0, 0.0, 1.0, 1.0)


def need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref/libaidw_ref.so not built (needs /root/reference at build time)")


def inputs(kind, m, n, seed):
    if kind == "clustered":
        xs, ys, zs = O.generate_clustered(m, seed=seed)
    else:
        xs, ys, zs = O.generate_points(m, UNIT, seed, 1 if kind == "planar" else 0)
    qx, qy = O.generate_queries(n, UNIT, seed + 1)
    return xs, ys, zs, qx, qy


def contract(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * max(span, 1e-300))))


@pytest.fixture(autouse=True)
def fp32_default():
    A.set_weight_precision("fp32")
    yield
    A.set_weight_precision("fp32")


@pytest.mark.parametrize("kind,m,n,k,levels", [
    ("uniform", 40_000, 3000, 10, (0.5, 1.0, 2.0, 3.0, 4.0)),
    ("clustered", 40_000, 3000, 10, (0.5, 1.0, 2.0, 3.0, 4.0)),
    ("planar", 25_000, 2000, 15, (0.5, 1.0, 2.0, 3.0, 4.0)),
    ("clustered", 30_000, 3000, 10, (1.0, 1.0, 3.0, 3.0, 4.0)),
    ("clustered", 30_000, 3000, 12, (2.0, 2.0, 1.0, 1.0, 3.0)),
])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_aidw_pipeline_matches_reference(kind, m, n, k, levels, precision):
    need_ref()
    xs, ys, zs, qx, qy = inputs(kind, m, n, 17)
    ref_pred, ref_alpha, _, ref_k = O.ref_run_pipeline(xs, ys, zs, qx, qy, mode=1, k=k,
                                                       levels=levels)
    A.set_weight_precision(precision)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(params=A.AidwParams(k=k, alpha_levels=levels)))
    assert out.k_effective == ref_k
    assert np.max(np.abs(out.result.alphas - ref_alpha) / ref_alpha) <= 1e-12
    tol = 1e-5 if precision == "fp32" else 2e-11
    assert contract(out.result.predicted, ref_pred, zs) <= tol


@pytest.mark.parametrize("alpha", [1.0, 2.0, 3.0, 4.0, 2.5])
def test_idw_pipeline_matches_reference(alpha):
    need_ref()
    xs, ys, zs, qx, qy = inputs("uniform", 30_000, 2500, 29)
    ref_pred, _, _, _ = O.ref_run_pipeline(xs, ys, zs, qx, qy, mode=0, alpha=alpha)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(mode="idw", alpha=alpha))
    assert np.all(out.result.alphas == alpha)
    assert contract(out.result.predicted, ref_pred, zs) <= 1e-5


@pytest.mark.parametrize("kind", ["uniform", "clustered"])
def test_bench_scale_data_matches_reference(kind):
    """BASELINE configs[2] / [3] data size (1M points: 3907 K4 tiles in 32
    data chunks, the bench's grid) against the reference on 4096 queries."""
    need_ref()
    xs, ys, zs, qx, qy = inputs(kind, 1_000_000, 4096, 42)
    ref_pred, ref_alpha, _, _ = O.ref_run_pipeline(xs, ys, zs, qx, qy, mode=1, k=10)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy),
                         A.RunConfig(params=A.AidwParams(k=10)))
    assert np.max(np.abs(out.result.alphas - ref_alpha) / ref_alpha) <= 1e-12
    assert contract(out.result.predicted, ref_pred, zs) <= 1e-5
