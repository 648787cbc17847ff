"""bench.py — interpolated points/s of the fused AIDW pipeline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1m|clustered|10k|100k|paper|dem] [--no-cpu-baseline]

A step = one full pass of the hot path (bbox -> grid build K1 -> query sort
-> kNN + alpha K2/K3 -> weighting K4 -> settle) over one batch: m = 1M data
points x n = 1M queries per rank (BASELINE.json configs[2]; weak scaling:
rank r interpolates slice r of an N*1M query set against the same 1M data,
replicated by an NCCL broadcast).  `value` times device-resident inputs with
CUDA events on the launching stream (L2 flushed between steps, max over
ranks); `e2e` times the public C-ABI call aidw_run_pipeline from pinned
host buffers (H2D + D2H inside).  `--impl reference` times the reference's
own CPU run_pipeline (oracle/_ref, compiled from /root/reference) on the
host cores with a deterministic query subsample, extrapolated exactly
(weighting and kNN cost are linear in n).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = (0.0, 0.0, 1.0, 1.0)
METRIC = "interpolated points/sec (kNN+weighting) at 1M x 1M"
CONFIGS = {
    "1m": dict(m=1_000_000, n=1_000_000, k=10, dist="uniform",
               workload="1M data x 1M queries per rank, uniform unit square, k=10 (BASELINE configs[2])"),
    "clustered": dict(m=1_000_000, n=1_000_000, k=10, dist="clustered",
                      workload="1M x 1M per rank, 20 Gaussian blobs sigma=0.03, k=10 (BASELINE configs[3])"),
    "10k": dict(m=10_000, n=10_000, k=10, dist="uniform",
                workload="10K x 10K uniform, k=10 (BASELINE configs[0], the reference's serial CPU case)"),
    "100k": dict(m=100_000, n=100_000, k=10, dist="uniform",
                 workload="100K x 100K uniform, k=10 (BASELINE configs[1])"),
    "paper": dict(m=1_024_000, n=1_024_000, k=10, dist="uniform",
                  workload="1000K x 1000K uniform (the paper's rung, 1K = 1024; SURVEY §8d), k=10"),
    "dem": dict(m=4_000_000, n=4096 * 4096, k=15, dist="lattice",
                workload="4M planar data x 4096^2 raster lattice, k=15 (BASELINE configs[4])"),
}


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        p.update(hbm_gbs=float(j.get("hbm_gbs", p["hbm_gbs"])),
                 sm_max_mhz=float(j.get("sm_max_mhz", p["sm_max_mhz"])), source="measured")
    return p


def k4_traffic(cfg):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K4 launch from the
    latest committed `ncu --set full` capture of the bench config (or None)."""
    import glob
    if cfg is not CONFIGS["1m"]:
        return None
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k4_traffic.json")))
    if not paths:
        return None
    with open(paths[-1]) as f:
        return json.load(f).get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/aidw_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            return None
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        busy = [s for s in sm if s > 0.5 * (max(mx) if mx else 1965)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def lattice_box(A, data, world):
    """cmd_raster's lattice box (bbox of the data, cli.hpp:495), stretched
    north by `world` so rank r owns rows [4096 r, 4096 (r + 1)) (weak scaling)."""
    bb = A.compute_bbox(data)
    return (bb.min_x, bb.min_y, bb.max_x, bb.min_y + (bb.max_y - bb.min_y) * world)


def make_inputs(A, cfg, world, rank):
    m, n = cfg["m"], cfg["n"]
    if cfg["dist"] == "clustered":
        data = A.generate_clustered(m, seed=42)
        allq = A.generate_clustered(n * world, seed=43, with_values=False)
    elif cfg["dist"] == "lattice":
        data = A.generate_random_points(m, UNIT, 42, "planar")
        allq = A.raster_lattice(4096, 4096 * world, lattice_box(A, data, world))
    else:
        data = A.generate_random_points(m, UNIT, 42)
        allq = A.generate_random_queries(n * world, UNIT, 43)
    from paper_1601_05904_b200.shard import shard_range
    lo, hi = shard_range(n * world, world, rank)
    return data, A.PointSet(allq.xs[lo:hi].copy(), allq.ys[lo:hi].copy())


def reference_cpu(cfg, data, queries, target_s=8.0, workers=0):
    """Time the reference's own cli::run_pipeline (oracle/_ref) on the host
    cores: full data, a deterministic strided query subsample sized for
    ~target_s of weighting; extrapolate kNN + weighting linearly in n."""
    import oracle as O
    if not O.ref_available():
        return None
    n = queries.count()
    threads = O.ref_hardware_threads() if workers == 0 else workers
    bb = (min(data.xs.min(), queries.xs.min()), min(data.ys.min(), queries.ys.min()),
          max(data.xs.max(), queries.xs.max()), max(data.ys.max(), queries.ys.max()))
    area = (bb[2] - bb[0]) * (bb[3] - bb[1])
    probe = max(1, n // 4000)
    qs = slice(0, n, probe)
    t = time.perf_counter()
    _, _, tm, _ = O.ref_run_pipeline(data.xs, data.ys, data.zs, queries.xs[qs], queries.ys[qs],
                                     k=cfg["k"], area=area, workers=workers)
    per_q = (tm[1] + tm[2]) / 1e3 / max(1, queries.xs[qs].size)
    n_s = int(min(n, max(256, target_s / max(per_q, 1e-9))))
    stride = max(1, n // n_s)
    qs = slice(0, n, stride)
    ns = queries.xs[qs].size
    _, _, tm, _ = O.ref_run_pipeline(data.xs, data.ys, data.zs, queries.xs[qs], queries.ys[qs],
                                     k=cfg["k"], area=area, workers=workers)
    wall = time.perf_counter() - t
    full_ms = tm[0] + (tm[1] + tm[2]) * (n / ns)
    return {"value": n / (full_ms / 1e3), "unit": "points/s", "cores": threads,
            "kind": "reference", "full_ms": full_ms, "timings_ms": tm.tolist(),
            "sample": (f"reference cli::run_pipeline (oracle/_ref, -O3 x86-64-v4 AVX-512, "
                       f"workers={threads}) on all {data.count()} data points and every "
                       f"{stride}th query ({ns} of {n}); build timed in full, kNN+weighting "
                       f"scaled by n/{ns}; {wall:.1f} s of CPU work")}


def run_reference_arm(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import paper_1601_05904_b200 as A
    data, queries = make_inputs(A, cfg, 1, 0)
    values, ms = [], []
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    base = None
    for i in range(args.warmup + args.steps):
        r = reference_cpu(cfg, data, queries, target_s=min(8.0, budget))
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable":
                              "oracle/_ref/libaidw_ref.so not built (reference not compiled)"}))
            return 0
        if i >= args.warmup:
            values.append(r["value"])
            ms.append(r["full_ms"])
            base = r
    value = statistics.median(values)
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(ms),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seeds 42/43)",
            "config": {"workload": cfg["workload"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"],
                       "parallelism": f"cpu threads x{base['cores']}"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": base["cores"],
                             "kind": "reference", "sample": base["sample"]},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="1m", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1601_05904_b200 as A

    world, rank, local = dist_env()
    # AIDW_BENCH_SHARED_DEVICE=1 (test hook): every rank on device 0 with the
    # gloo backend, so the multi-rank path runs end to end on a one-GPU box
    shared = os.environ.get("AIDW_BENCH_SHARED_DEVICE") == "1"
    local = 0 if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    name, sms = A.device_info()
    data, queries = make_inputs(A, cfg, world, rank)
    m, n = data.count(), queries.count()

    from paper_1601_05904_b200 import shard

    # data: rank 0's copy replicated over NVLink (NCCL broadcast)
    d_data = torch.from_numpy(np.stack([data.xs, data.ys, data.zs])).to(dev)
    shard.replicate(d_data, dist if world > 1 else None)
    d_q = torch.from_numpy(np.stack([queries.xs, queries.ys])).to(dev)
    d_pred = torch.empty(n, dtype=torch.float64, device=dev)
    d_alpha = torch.empty(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    dx, dy, dz = (d_data[i].data_ptr() for i in range(3))
    qx, qy = d_q[0].data_ptr(), d_q[1].data_ptr()

    # global bbox(data ∪ all queries): per-rank device reduce + all-reduce
    bb = shard.global_bbox(A.compute_bbox_device(dx, dy, m, qx, qy, n, sp),
                           dist if world > 1 else None, device=dev)
    rc = A.RunConfig(params=A.AidwParams(k=cfg["k"]), bbox=tuple(float(v) for v in bb))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    lattice = cfg["dist"] == "lattice"
    if lattice:  # cmd_raster: the lattice rows of this rank are generated in HBM each step
        lbox = lattice_box(A, data, world)

    def step():
        if lattice:
            A.raster_lattice_device(4096, 4096 * world, lbox, qx, qy, 4096 * rank, 4096, sp)
        return A.run_pipeline_device(dx, dy, dz, m, qx, qy, n, rc, d_pred.data_ptr(),
                                     d_alpha.data_ptr(), sp)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stats = []
    l0 = A.kernel_launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (256 MiB write), not timed
            starts[i].record(stream)
            stats.append(step())
            ends[i].record(stream)
        barrier()
    launches = A.kernel_launch_count() - l0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = allmax(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = world * n / (ms_per_step / 1e3)

    # roofline of the dominant kernel (K4): live CUDA-event duration of the
    # weight_fp32_kernel launch inside each timed step
    pk = peaks()
    f_mhz = pk["sm_max_mhz"]
    k4_ms = statistics.median(s["weight_kernel_ms"] for s in stats)
    pairs = m * n
    peak_gpairs = sms * 8 * f_mhz * 1e6 / 1e9  # 2 MUFU / pair, 16 MUFU / clk / SM
    achieved = pairs / (k4_ms / 1e3) / 1e9
    knn_ms = statistics.median(s["knn_kernel_ms"] for s in stats)
    cand = stats[-1]["knn_candidates"]  # points K2 actually scanned (after cell pruning)
    ref_cand = stats[-1]["knn_ref_candidates"]  # points the reference scans (final-level blocks)
    # SURVEY §8d algorithmic bytes: 16 B query + 16 B per reference candidate + outputs
    knn_bytes = n * (16 + 8 + 8 + 4 + 4) + 16 * ref_cand
    build_ms = statistics.median(s["build_ms"] for s in stats)
    build_bytes = 64 * m + 8 * (m // 4 + 1)  # factor-4 grid: ~m/4 cells (SURVEY §8 grid table)
    a4 = stats[-1]["alpha4_queries"]
    # Pipe roofline of the executed formula mix (K4 far-tile forms):
    # per SM and clock the FMA pipe retires 128 FP32 ops (FFMA2 = 2) and the
    # XU pipe 16 MUFU ops; a class is bound by the slower of the two.
    #   recipe (alpha == 4): 3 (d2) + 1 (d2^2) + 2.5 (pair/single sums) = 6.5
    #     FP32 + 0.75 MUFU per pair (two of every four points share one rcp)
    #   general: G1 6 FP32 + 2 MUFU (lg2, ex2), G2 14 FP32 + 1 MUFU (ex2 as a
    #     degree-5 polynomial); G1 / G2 split ~1:1 by coordinate hash
    clk_recipe = max(6.5 / 128, 0.75 / 16)
    clk_general = max(0.5 * (6 + 14) / 128, 0.5 * (2 + 1) / 16)
    clk_mix = (a4 * clk_recipe + (n - a4) * clk_general) / n
    peak_mix = sms * f_mhz * 1e6 / clk_mix / 1e9
    peak_general = sms * f_mhz * 1e6 / clk_general / 1e9

    # general-alpha path forced (every query on exp2/log2), reported separately
    A.set_alpha4_recipe(False)
    gen = []
    for _ in range(2):
        flush.zero_()
        gen.append(step())
    A.set_alpha4_recipe(True)
    k4g_ms = statistics.median(s["weight_kernel_ms"] for s in gen)
    torch.cuda.synchronize()

    # e2e through the public C-ABI with pinned host buffers
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in
           dict(dx=data.xs, dy=data.ys, dz=data.zs, qx=queries.xs, qy=queries.ys).items()}
    hd = A.PointSet(pin["dx"].numpy(), pin["dy"].numpy(), pin["dz"].numpy())
    hq = A.PointSet(pin["qx"].numpy(), pin["qy"].numpy())
    hcfg = A.RunConfig(params=A.AidwParams(k=cfg["k"]), bbox=rc.bbox)
    raster_e2e = lattice and world == 1
    if raster_e2e:
        # the public raster call: host data in, raster out (lattice in HBM)
        rcfg = A.RunConfig(params=A.AidwParams(k=cfg["k"]))

        def e2e_call():
            return A.run_raster(hd, 4096, 4096, rcfg, with_alpha=False)
    else:
        # results land in pinned host buffers (the C-ABI writes caller memory)
        pout = (torch.empty(n, dtype=torch.float64).pin_memory().numpy(),
                torch.empty(n, dtype=torch.float64).pin_memory().numpy())

        def e2e_call():
            return A.run_pipeline(hd, hq, hcfg, out=pout)
    e2e_call()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_call()
    barrier()
    e2e_s = allmax((time.perf_counter() - t0) / args.e2e_steps)
    e2e_value = world * n / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = reference_cpu(cfg, data, queries)
        if cpu is None:
            cpu = {"value": None, "unit": "points/s", "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not available"}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 weighting / f64 grid+kNN+alpha",
            "data": "synthetic (reference mt19937_64 generator, seeds 42/43)",
            "config": {"workload": cfg["workload"], "m": m, "n_per_rank": n, "k": cfg["k"],
                       "parallelism": f"query-sharded x{world}, data replicated (NCCL broadcast)",
                       "l2": "flushed between timed steps (256 MiB write)",
                       "device": name, "sms": sms},
            "roofline": {"bound": "fp32+mufu pipes", "kernel": "weight_fp32_kernel (K4)",
                         "achieved": achieved, "peak": peak_mix, "unit": "Gpair/s",
                         "frac": achieved / peak_mix, "traffic": k4_traffic(cfg),
                         "peak_def": f"{sms} SMs x {f_mhz:.0f} MHz ({pk['source']} sm_max_mhz) / "
                                     f"{clk_mix:.4f} SM-clk per pair: executed mix of the "
                                     f"alpha=4 recipe ({a4} queries; FMA-bound 6.5 FP32 + "
                                     f"0.75 MUFU) and general alpha (MUFU-bound 10 FP32 + "
                                     f"1.5 MUFU) far-tile forms; 128 FP32 + 16 MUFU per SM-clk",
                         "frac_vs_2mufu_roofline": achieved / peak_gpairs,
                         "fp32_view": {  # the same bound as FP32 op throughput
                             "unit": "TFLOP/s (FP32 ops, FFMA = 1)",
                             "ops_per_pair": (a4 * 6.5 + (n - a4) * 10.0) / n,
                             "achieved": achieved * 1e9 * (a4 * 6.5 + (n - a4) * 10.0) / n / 1e12,
                             "peak": sms * 128 * f_mhz * 1e6 / 1e12,
                             "frac": achieved * 1e9 * (a4 * 6.5 + (n - a4) * 10.0) / n /
                                     (sms * 128 * f_mhz * 1e6)},
                         "alpha4_recipe_queries": a4, "pairs_per_launch": pairs,
                         "k4_ms": k4_ms},
            "roofline_general_alpha": {"bound": "fp32+mufu pipes (MUFU-bound)",
                                       "achieved": pairs / (k4g_ms / 1e3) / 1e9,
                                       "peak": peak_general, "unit": "Gpair/s",
                                       "frac": pairs / (k4g_ms / 1e3) / 1e9 / peak_general,
                                       "frac_vs_2mufu_roofline":
                                           pairs / (k4g_ms / 1e3) / 1e9 / peak_gpairs,
                                       "k4_ms": k4g_ms},
            "stages": {
                "build_ms": build_ms,
                "knn_kernel_ms": knn_ms,
                "knn_hbm": {"bytes": knn_bytes, "achieved_gbs": knn_bytes / (knn_ms / 1e3) / 1e9,
                            "peak_gbs": pk["hbm_gbs"],
                            "frac": knn_bytes / (knn_ms / 1e3) / 1e9 / pk["hbm_gbs"],
                            "candidates_reference": ref_cand, "candidates_scanned": cand},
                "build_hbm": {"bytes": build_bytes,
                              "achieved_gbs": build_bytes / (build_ms / 1e3) / 1e9,
                              "frac": build_bytes / (build_ms / 1e3) / 1e9 / pk["hbm_gbs"]},
                "weight_ms": k4_ms, "interp_ms": statistics.median(s["interp_ms"] for s in stats),
            },
            "e2e": {"value": e2e_value, "unit": "points/s",
                    "api": "aidw_run_raster (C-ABI)" if raster_e2e else "aidw_run_pipeline (C-ABI)",
                    "h2d_bytes_per_step": 24 * m + (0 if raster_e2e else 16 * n),
                    "d2h_bytes_per_step": (8 if raster_e2e else 16) * n,
                    "s_per_step": e2e_s},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
