import sys, os
sys.path.insert(0, '.')
import paper_1601_05904_b200 as A
UNIT = (0.0, 0.0, 1.0, 1.0)
for m, n in ((20_000_000, 20_000), (4_000_000, 50_000), (1_000_000, 100_000)):
    data = A.generate_random_points(m, UNIT, 5)
    q = A.generate_random_queries(n, UNIT, 6)
    for _ in range(2):
        out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    print(os.environ.get("AIDW_K4_VARIANT", "0"), m, n, round(out.stats["weight_kernel_ms"], 2), round(m * n / out.stats["weight_kernel_ms"] / 1e9, 3), "Tpair/s", flush=True)
