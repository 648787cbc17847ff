import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1601_05904_b200 as A
for m, n in ((10_000, 10_000), (100_000, 100_000)):
    d = A.generate_random_points(m, (0, 0, 1, 1), 42); q = A.generate_random_queries(n, (0, 0, 1, 1), 43)
    dev = torch.device("cuda", 0)
    D = torch.from_numpy(np.stack([d.xs, d.ys, d.zs])).to(dev); Q = torch.from_numpy(np.stack([q.xs, q.ys])).to(dev)
    P = torch.empty(n, dtype=torch.float64, device=dev); AL = torch.empty(n, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    bb = A.compute_bbox_device(D[0].data_ptr(), D[1].data_ptr(), m, Q[0].data_ptr(), Q[1].data_ptr(), n, s.cuda_stream)
    for withbb in (False, True):
        cfg = A.RunConfig(params=A.AidwParams(k=10), bbox=tuple(float(v) for v in bb) if withbb else None).c()
        for i in range(8):
            st = A.run_pipeline_device(D[0].data_ptr(), D[1].data_ptr(), D[2].data_ptr(), m, Q[0].data_ptr(), Q[1].data_ptr(), n, cfg, P.data_ptr(), AL.data_ptr(), s.cuda_stream)
        print("bbox given" if withbb else "bbox computed", m, n, {k: round(v, 3) for k, v in st.items() if k.endswith('_ms')}, file=sys.stderr)
