"""One FP64-mode pipeline pass at a bench config, for ncu (weight_fp64_kernel).

    python tools/profile_fp64.py [--config 100k] [--variant blocked|naive]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1601_05904_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="100k", choices=sorted(bench.CONFIGS))
ap.add_argument("--variant", default="blocked", choices=["blocked", "naive"])
ap.add_argument("--passes", type=int, default=1)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
data, q = bench.lib_inputs(A, cfg)
A.set_weight_precision("fp64")
for _ in range(args.passes):
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=cfg["k"]), variant=args.variant))
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in out.stats.items()})
