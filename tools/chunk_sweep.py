"""K4 time vs the data-chunk granularity (AIDW_K4_CHUNK_TILES) for small data
sets at small and large query counts (GPU box)."""
import sys
sys.path.insert(0, '.')
import paper_1601_05904_b200 as A

UNIT = (0.0, 0.0, 1.0, 1.0)
for m, n in ((10_000, 10_000), (10_000, 1_000_000), (50_000, 50_000), (50_000, 1_000_000)):
    data = A.generate_random_points(m, UNIT, 5)
    q = A.generate_random_queries(n, UNIT, 6)
    for _ in range(3):
        out = A.run_pipeline(data, q, A.RunConfig(params=A.AidwParams(k=10)))
    print(m, n, round(out.stats["weight_kernel_ms"], 3), "ms", flush=True)
