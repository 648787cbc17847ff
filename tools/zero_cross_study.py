"""Contract error of the FP32 weighting on zero-mean white-noise value
fields (z uniform in [-s/2, s/2], predictions near 0 relative to the span):
error = |got - ref| / max(|ref|, 1e-3 span) against the C oracle, per K4
engine (run once per AIDW_K4_ENGINE setting)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1601_05904_b200 as A  # noqa: E402

UNIT = (0.0, 0.0, 1.0, 1.0)
for m in (10_000, 80_000, 300_000):
    data = A.generate_random_points(m, UNIT, 9)
    for name, zs in (("white+-", (data.zs - 0.5) * 1e30), ("white+", data.zs)):
        q = A.generate_random_queries(1000, UNIT, 10)
        out = A.run_pipeline(A.PointSet(data.xs, data.ys, zs), q, A.RunConfig(params=A.AidwParams(k=10)))
        ref = O.pipeline(data.xs, data.ys, zs, q.xs, q.ys, k=10, variant=1)
        span = zs.max() - zs.min()
        err = np.abs(out.result.predicted - ref["pred"]) / np.maximum(np.abs(ref["pred"]), 1e-3 * span)
        i = int(np.argmax(err))
        print(f"engine={A.weight_engine(m):11s} m={m:7d} {name:8s} max err {err.max():.2e} "
              f"(abs {np.abs(out.result.predicted - ref['pred']).max() / span:.2e} of span) "
              f"p99 {np.quantile(err, 0.99):.2e} alpha {ref['alpha'][i]:.3f}")
