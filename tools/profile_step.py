"""One warm-up + one measured fused pipeline pass at a bench config, for ncu.

    python tools/profile_step.py [--config 1m] [--general]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1601_05904_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1m", choices=sorted(bench.CONFIGS))
ap.add_argument("--general", action="store_true", help="force the general exp2/log2 path")
ap.add_argument("--passes", type=int, default=2)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
data, q = bench.lib_inputs(A, cfg)
if args.general:
    A.set_alpha4_recipe(False)
for i in range(args.passes):
    out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=cfg["k"])))
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in out.stats.items()})
