"""K4 accuracy study at bench sizes (test infrastructure, run on the GPU box).

    python tests/accuracy_study.py [--config 1m|clustered|100k] [--general] [--sample 1024]

Runs the fused pipeline, then recomputes a stratified query sample with the
C oracle's FP64 blocked predictor (oracle/aidw_oracle.c, the reference's
predict_blocked_fast arithmetic) using the GPU's alphas, and prints the
contract error |gpu - ref| / max(|ref|, 1e-3 * hull span) (max, p99, median)
— the margin the FP32 kernel keeps against the 1e-5 tolerance.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_1601_05904_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1m", choices=["1m", "clustered", "100k"])
ap.add_argument("--general", action="store_true")
ap.add_argument("--sample", type=int, default=1024)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
data, q = bench.lib_inputs(A, cfg)
if args.general:
    A.set_alpha4_recipe(False)
out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=cfg["k"])))
pred, alpha = out.result.predicted, out.result.alphas
n = len(pred)
rng = np.random.default_rng(1)
sample = np.sort(rng.choice(n, min(args.sample, n), replace=False))
ref = O.predict_with_alphas(q.xs[sample], q.ys[sample], data.xs, data.ys, data.zs,
                            alpha[sample], 1)
span = data.zs.max() - data.zs.min()
err = np.abs(pred[sample] - ref) / np.maximum(np.abs(ref), 1e-3 * span)
print(json.dumps({"config": args.config, "general": args.general, "sample": len(sample),
                  "rfar": os.environ.get("AIDW_K4_RFAR", "default"),
                  "max": float(err.max()), "p99": float(np.quantile(err, 0.99)),
                  "median": float(np.median(err)),
                  "weight_ms": out.stats.get("weight_kernel_ms")}))
