"""Large-size sanity runs (index-width / memory paths): many queries against
small data, many data points against few queries; spot-checked against the
C oracle on a query sample."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1601_05904_b200 as A  # noqa: E402

UNIT = (0.0, 0.0, 1.0, 1.0)
for m, n in ((100_000, 40_000_000), (20_000_000, 20_000)):
    data = A.generate_random_points(m, UNIT, 5)
    q = A.generate_random_queries(n, UNIT, 6)
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 64, replace=False))
    idx[-1] = n - 1  # the last query too
    ref = O.predict_with_alphas(q.xs[idx], q.ys[idx], data.xs, data.ys, data.zs,
                                out.result.alphas[idx], 1)
    span = data.zs.max() - data.zs.min()
    err = np.max(np.abs(out.result.predicted[idx] - ref) / np.maximum(np.abs(ref), 1e-3 * span))
    print(f"m={m} n={n}: weight {out.stats['weight_kernel_ms']:.1f} ms, "
          f"knn {out.stats['knn_kernel_ms']:.2f} ms, sample err {err:.2e}", flush=True)
    assert err <= 1e-5 and np.all(np.isfinite(out.result.predicted))
print("large sizes ok")
