"""Generate tests/golden/*.npz from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libaidw_ref.so, compiled
from /root/reference/proj/include by `make -C oracle ref`).  The fixtures are
committed so the GPU box — where /root/reference does not exist — can check
both the C restatement and the CUDA path against reference outputs.

    python tests/golden/make_golden.py

Every fixture records the reference call that produced it.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
UNIT = (0.0, 0.0, 1.0, 1.0)
LEVELS = (0.5, 1.0, 2.0, 3.0, 4.0)


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def gen_fixture():
    """generate.hpp:45-95 — seeds/bboxes/rules used across the reference tests."""
    out = {}
    cases = [(500, UNIT, 42, 0), (500, UNIT, 42, 1), (500, UNIT, 42, 2),
             (300, (-3.0, 5.0, 17.0, 25.0), 1003, 0), (100, (0.0, 0.0, 10.0, 10.0), 1, 0)]
    for i, (cnt, bb, seed, rule) in enumerate(cases):
        xs, ys, zs = O.ref_generate_points(cnt, bb, seed, rule)
        out[f"p{i}_args"] = np.array([cnt, *bb, seed, rule], dtype=np.float64)
        out[f"p{i}_x"], out[f"p{i}_y"], out[f"p{i}_z"] = xs, ys, zs
    qx, qy = O.ref_generate_queries(400, UNIT, 43)
    out["q_args"] = np.array([400, *UNIT, 43], dtype=np.float64)
    out["q_x"], out["q_y"] = qx, qy
    save("generate", **out)


def grid_fixture():
    """build_index on the test_grid.cpp:204-274 instance (2000 pts, seed 21, factor 4)
    and the :172-202 instance (1000 pts, seed 7, width 1/15.5)."""
    out = {}
    for tag, (cnt, seed, width) in {"a": (2000, 21, None), "b": (1000, 7, 1.0 / 15.5)}.items():
        xs, ys, zs = O.ref_generate_points(cnt, UNIT, seed, 0)
        if width is None:
            cfg5 = O.ref_grid_config(xs, ys, np.empty(0), np.empty(0), 4.0)
        else:
            cfg = O.make_grid_config(np.array(UNIT), width)
            cfg5 = np.array([cfg.cell_width, cfg.n_col, cfg.n_row, cfg.min_x, cfg.min_y])
        ids, cs, sx, sy = O.ref_build_index(xs, ys, cfg5)
        out.update({f"{tag}_x": xs, f"{tag}_y": ys, f"{tag}_cfg": cfg5, f"{tag}_ids": ids,
                    f"{tag}_cell_start": cs, f"{tag}_sx": sx, f"{tag}_sy": sy})
    save("grid", **out)


def knn_fixture():
    """knn_stage (grid engine, factor 4 / factor 1) — test_knn.cpp:202-247."""
    out = {}
    specs = {
        "std": (2000, 3, 200, 4, 4.0, (1, 5, 15)),
        "tiny": (300, 8, 50, 9, 1.0, (1, 7, 64)),
        "exh": (5, 2, 7, 77, 4.0, (64,)),
    }
    for tag, (m, ds, n, qs, factor, ks) in specs.items():
        xs, ys, zs = O.ref_generate_points(m, UNIT, ds, 0)
        qx, qy = O.ref_generate_queries(n, UNIT, qs)
        out.update({f"{tag}_x": xs, f"{tag}_y": ys, f"{tag}_qx": qx, f"{tag}_qy": qy,
                    f"{tag}_factor": np.array([factor]), f"{tag}_ks": np.array(ks)})
        for k in ks:
            d2, avg, exh, lens = O.ref_knn_stage(qx, qy, xs, ys, k, engine=0, factor=factor)
            out.update({f"{tag}_k{k}_d2": d2, f"{tag}_k{k}_avg": avg,
                        f"{tag}_k{k}_exh": exh, f"{tag}_k{k}_len": lens})
    # shifted domain with queries past the data hull (acceptance.cpp:84-92 pattern)
    box = (-3.0, 5.0, 17.0, 25.0)
    xs, ys, zs = O.ref_generate_points(1500, box, 1003, 0)
    qx, qy = O.ref_generate_queries(150, (-5.0, 3.0, 19.0, 27.0), 900003)
    d2, avg, exh, lens = O.ref_knn_stage(qx, qy, xs, ys, 10, engine=0, factor=2.0)
    out.update({"shift_x": xs, "shift_y": ys, "shift_qx": qx, "shift_qy": qy, "shift_d2": d2,
                "shift_avg": avg})
    save("knn", **out)


def adaptive_fixture():
    """adaptive_alpha over random (r_obs, m, area) — test_adaptive.cpp:201-219 pattern."""
    rng = np.random.default_rng(2024)
    r_obs = 3.0 * rng.random(400)
    m = 1 + rng.integers(0, 5000, 400)
    area = 0.5 + 99.5 * rng.random(400)
    rec = np.array([O.ref_adaptive_alpha(r, int(mm), a, k=4, levels=LEVELS)
                    for r, mm, a in zip(r_obs, m, area)])
    jumbled = (3.0, 0.5, 4.0, 1.0, 2.0)
    rec_j = np.array([O.ref_adaptive_alpha(r, int(mm), a, k=4, levels=jumbled, r_min=0.5)
                      for r, mm, a in zip(r_obs, m, area)])
    save("adaptive", r_obs=r_obs, m=m, area=area, rec=rec, rec_jumbled=rec_j,
         jumbled=np.array(jumbled))


def predict_fixture():
    """Weighting: idw / aidw, naive and blocked, reference outputs."""
    out = {}
    # test_interpolate.cpp:117-132 — 1000 x 1000, alpha 2, seeds 40/41
    xs, ys, zs = O.ref_generate_points(1000, UNIT, 40, 0)
    qx, qy = O.ref_generate_queries(1000, UNIT, 41)
    pn, _ = O.ref_predict_all(xs, ys, zs, qx, qy, mode=0, variant=0, alpha=2.0, workers=8)
    pb, _ = O.ref_predict_all(xs, ys, zs, qx, qy, mode=0, variant=1, alpha=2.0, workers=8)
    pp, _ = O.ref_predict_all(xs, ys, zs, qx, qy, mode=0, variant=1, pinned=True, alpha=2.0,
                              workers=8)
    out.update(idw_x=xs, idw_y=ys, idw_z=zs, idw_qx=qx, idw_qy=qy, idw_naive=pn,
               idw_blocked=pb, idw_pinned=pp)
    # AIDW, radial values, k=15, grid engine — 3000 x 500
    xs, ys, zs = O.ref_generate_points(3000, UNIT, 50, 2)
    qx, qy = O.ref_generate_queries(500, (-0.1, -0.1, 1.1, 1.1), 51)
    pn, an = O.ref_predict_all(xs, ys, zs, qx, qy, mode=1, variant=0, k=15, workers=8)
    pb, ab = O.ref_predict_all(xs, ys, zs, qx, qy, mode=1, variant=1, k=15, workers=8)
    out.update(aidw_x=xs, aidw_y=ys, aidw_z=zs, aidw_qx=qx, aidw_qy=qy, aidw_naive=pn,
               aidw_blocked=pb, aidw_alpha=an, aidw_alpha_b=ab)
    # degenerate weights -> nearest value (test_interpolate.cpp:251-266)
    dx = np.array([0.0, 1.0e-160]); dy = np.zeros(2); dz = np.array([3.0, 9.0])
    pq = np.array([4.0e-161]); pqy = np.zeros(1)
    pdn, _ = O.ref_predict_all(dx, dy, dz, pq, pqy, mode=0, variant=0, alpha=2.0)
    pdb, _ = O.ref_predict_all(dx, dy, dz, pq, pqy, mode=0, variant=1, alpha=2.0)
    out.update(degen_naive=pdn, degen_blocked=pdb)
    save("predict", **out)


def pipeline_fixture():
    """Config 1 (BASELINE.json configs[0]): 10K x 10K uniform, k=10, run_pipeline
    (aidw, grid, blocked and naive), plus its grid-kNN lists."""
    xs, ys, zs = O.ref_generate_points(10000, UNIT, 42, 0)
    qx, qy = O.ref_generate_queries(10000, UNIT, 43)
    pb, ab, _, keff = O.ref_run_pipeline(xs, ys, zs, qx, qy, variant=1, k=10, workers=8)
    pn, an, _, _ = O.ref_run_pipeline(xs, ys, zs, qx, qy, variant=0, k=10, workers=8)
    d2, avg, exh, lens = O.ref_knn_stage(qx, qy, xs, ys, 10, engine=0, workers=8)
    save("pipeline10k", pred_blocked=pb, alpha=ab, pred_naive=pn, alpha_naive=an, d2=d2,
         avg=avg, k_eff=np.array([keff]), seeds=np.array([42, 43]))
    # clustered data (harness generator) at 20K x 5K, k=10
    cx, cy, cz = O.generate_clustered(20000, seed=42)
    cqx, cqy = O.generate_clustered(5000, seed=43, with_values=False)
    pb, ab, _, _ = O.ref_run_pipeline(cx, cy, cz, cqx, cqy, variant=1, k=10, workers=8)
    d2, avg, exh, lens = O.ref_knn_stage(cqx, cqy, cx, cy, 10, engine=0, workers=8)
    save("clustered", x=cx, y=cy, z=cz, qx=cqx, qy=cqy, pred_blocked=pb, alpha=ab, d2=d2,
         avg=avg)


if __name__ == "__main__":
    if not O.ref_available():
        sys.exit("oracle/_ref/libaidw_ref.so missing: run `make -C oracle ref` first")
    gen_fixture()
    grid_fixture()
    knn_fixture()
    adaptive_fixture()
    predict_fixture()
    pipeline_fixture()
