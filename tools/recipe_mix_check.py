"""Recipe-class mixing check (GPU box): AIDW with alpha levels saturating at
exactly 1, 2, 3 and 4 on clustered data, so warps of the alpha = 4 / 2 / 1 / 3
recipe regions and the general region meet; prints the worst contract errors
against the C oracle.  Run it against a library built with
-DAIDW_K4_FORCE_MIXED=1 (tools/build_variant.sh, AIDW_LIB_PATH) to force
every recipe warp through the per-slot mixed form — the errors must not move."""
import sys; sys.path.insert(0,'.')
import numpy as np, oracle as O, paper_1601_05904_b200 as A
def pe(got, ref, zs):
    span = float(np.max(zs) - np.min(zs))
    return np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * span)
xs, ys, zs = O.generate_clustered(30_000, seed=11)
qx, qy = O.generate_queries(3000, (0.0, 0.0, 1.0, 1.0), 12)
for lv in [(2.0, 2.0, 3.0, 4.0, 4.0), (1.0, 1.0, 3.0, 3.0, 4.0), (1.0, 1.0, 2.0, 2.0, 3.0),
           (4.0,) * 5, (2.0,) * 5, (1.0,) * 5, (3.0,) * 5]:
    p = A.AidwParams(k=10, alpha_levels=lv)
    ref = O.pipeline(xs, ys, zs, qx, qy, k=10, variant=1, levels=lv)
    out = A.run_pipeline(A.PointSet(xs, ys, zs), A.PointSet(qx, qy), A.RunConfig(params=p))
    e = pe(out.result.predicted, ref["pred"], zs)
    al = ref["alpha"]
    bad = np.argsort(e)[-5:]
    print(lv, "max", e.max(), "nbad", (e>1e-5).sum(), "bad alphas", al[bad], "d2min", ref["d2"][bad,0], flush=True)
