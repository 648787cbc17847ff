import sys, time
sys.path.insert(0, '.')
import bench, paper_1601_05904_b200 as A
for cfgname, variant in [(c, v) for c in sys.argv[1:] or ["100k"] for v in ("blocked", "naive")]:
    cfg = bench.CONFIGS[cfgname]
    data, q = bench.lib_inputs(A, cfg)
    A.set_weight_precision("fp64")
    for i in range(2):
        out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=cfg["k"]), variant=variant))
    print(cfgname, variant, "fp64 weight_ms", round(out.stats["weight_kernel_ms"], 2), flush=True)
    A.set_weight_precision("fp32")
