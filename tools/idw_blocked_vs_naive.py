"""The reference's test_interpolate 1000 x 1000 instance (blocked vs naive
<= 1e-6 relative): error distribution of the FP32 kernel at alpha = 2."""
import sys; sys.path.insert(0, '.')
import numpy as np, oracle as O, paper_1601_05904_b200 as A
xs, ys, zs = O.generate_points(1000, (0.0, 0.0, 1.0, 1.0), 40, 0)
qx, qy = O.generate_queries(1000, (0.0, 0.0, 1.0, 1.0), 41)
ref = O.predict_with_alphas(qx, qy, xs, ys, zs, np.full(1000, 2.0), 0)
for rec in (True, False):
    A.set_alpha4_recipe(rec)
    got = A.idw_predict_all(A.PointSet(qx, qy), A.PointSet(xs, ys, zs), 2.0).predicted
    e = np.abs(got - ref) / np.abs(ref)
    i = np.argsort(e)[-5:]
    print("recipe", rec, "max", e.max(), "n>1e-6", (e > 1e-6).sum(), "p99", np.percentile(e, 99),
          "worst ref", ref[i], flush=True)
