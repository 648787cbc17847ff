"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the fused pipeline (FP32 and FP64 weighting, aidw and
idw), the drop-in batch calls, the raster path, a crowded-cell grid, the recipe
classes (alpha = 1, 2, 3, 4, mixed warps), the per-call workspace reuse, and
the tensor-core K4 engine (m >= 64K) with its side-stream CUDA-core launch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1601_05904_b200 as A  # noqa: E402

UNIT = (0.0, 0.0, 1.0, 1.0)
data = A.generate_random_points(5000, UNIT, 1)
q = A.generate_random_queries(777, UNIT, 2)
A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
A.run_pipeline(data, q, A.RunConfig(mode="idw", alpha=2.0))
A.run_pipeline(data, q, A.RunConfig(mode="idw", alpha=1.0))
A.run_pipeline(data, q, A.RunConfig(mode="idw", alpha=3.0))
# recipe classes mixed with each other and with general alpha in one warp
A.run_pipeline(A.generate_clustered(8000, seed=5), q,
               A.RunConfig(params=A.AidwParams(k=10, alpha_levels=(1.0, 1.0, 2.0, 3.0, 4.0))))
A.set_weight_precision("fp64")
A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=15)))
A.set_weight_precision("fp32")
cl = A.generate_clustered(6000, seed=3)
A.run_pipeline(cl, A.generate_clustered(500, seed=4, with_values=False),
               A.RunConfig(params=A.AidwParams(k=10), knn_engine="brute"))
A.run_raster(data, 33, 21, A.RunConfig(params=A.AidwParams(k=15)))
xs = np.concatenate([np.full(5000, 0.5), np.random.default_rng(0).random(2000)])
ys = np.concatenate([np.full(5000, 0.5), np.random.default_rng(1).random(2000)])
zs = np.arange(7000, dtype=np.float64)
A.run_pipeline(A.PointSet(xs, ys, zs), q, A.RunConfig(params=A.AidwParams(k=10)))
# m >= 64K: the tensor-core K4 engine (recipe queries) beside the CUDA-core
# launch (general-alpha queries) on its side stream
big = A.generate_random_points(70_000, UNIT, 7)
A.run_pipeline(big, A.generate_random_queries(1500, UNIT, 8), A.RunConfig(params=A.AidwParams(k=10)))
A.run_pipeline(A.generate_clustered(70_000, seed=9), A.generate_clustered(1200, seed=10, with_values=False),
               A.RunConfig(params=A.AidwParams(k=10, alpha_levels=(1.0, 1.0, 2.0, 3.0, 4.0))))
print("sanitize run ok")
