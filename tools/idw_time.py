"""Constant-alpha IDW timing and accuracy (integer alpha 1-4 use the recipe
classes — one reciprocal or reciprocal square root per point — other alphas
the general lg2/ex2 form): K4 time at 1M x 1M, and the maximum
relative prediction error against the C oracle at 100K x 20K."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle as O
import paper_1601_05904_b200 as A

UNIT = (0.0, 0.0, 1.0, 1.0)
for alpha in (2.0, 1.0, 3.0, 4.0, 2.5):
    cfg = A.RunConfig(mode="idw", alpha=alpha, params=A.AidwParams(k=10))
    data = A.generate_random_points(1_000_000, UNIT, 5)
    q = A.generate_random_queries(1_000_000, UNIT, 6)
    for _ in range(2):
        out = A.run_pipeline(data, q, cfg)
    ms = out.stats["weight_kernel_ms"]
    xs, ys, zs = O.generate_points(100_000, UNIT, 7, 0)
    qx, qy = O.generate_queries(20_000, UNIT, 8)
    got = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy), cfg).result.predicted
    ref = O.predict_with_alphas(qx, qy, xs, ys, zs, np.full(qx.size, alpha), variant=1)
    err = float(np.max(np.abs(got - ref) / np.abs(ref)))
    print(f"alpha {alpha}: K4 {ms:.1f} ms at 1M x 1M; max rel err {err:.2e} at 100K x 20K", flush=True)
