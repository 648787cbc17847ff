"""bench.py — interpolated points/s of the fused AIDW pipeline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1m|clustered|stress|10k|100k|paper|dem]
                    [--scaling strong|weak] [--no-cpu-baseline] [--no-fp64]

A step = one full pass of the hot path (bbox -> grid build K1 -> query sort
-> kNN + alpha K2/K3 -> weighting K4 -> settle) over one batch.  Default
config: BASELINE.json configs[2], m = 1M data points x n = 1M queries,
uniform, k = 10.  At N > 1 the 1M queries are sharded over the ranks exactly
as configs[2] is written (strong scaling: value = n / max-rank time); every
rank holds the data, replicated from rank 0 by an NCCL broadcast, and the
global bbox comes from a 4-double all-reduce.  A weak-scaling figure (N x 1M
queries, 1M per rank) is reported beside it.  `value` times device-resident
inputs with CUDA events on the launching stream (L2 flushed between steps,
max over ranks); `e2e` times the public C-ABI call aidw_run_pipeline from
pinned host buffers (H2D + D2H inside); `fp64` is the same pipeline with the
FP64 weighting kernel (the reference's precision).

`--impl reference` times the reference's own CPU cli::run_pipeline
(oracle/_ref/libaidw_ref.so, compiled in place from /root/reference) on all
host threads, on inputs made by the reference's own generator — this arm
never loads the repo's library.  Each timed step is a full pass over all n
queries when K full passes fit AIDW_REF_BUDGET_S (default 300 s); otherwise
each step interpolates a fixed strided query sample and the line reports the
throughput measured on it (`cpu_baseline.sampled`).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
               workload="1M data x 1M queries, uniform unit square, k=10 (BASELINE configs[2])"),
    "clustered": dict(m=1_000_000, n=1_000_000, k=10, dist="clustered",
                      workload="1M x 1M, 20 Gaussian blobs sigma=0.03, k=10 (BASELINE configs[3])"),
    "stress": dict(m=1_000_000, n=1_000_000, k=10, dist="stress",
                   workload="1M blob data (20 blobs, sigma=0.03) x 1M uniform queries, k=10 "
                            "(configs[3] stress variant: void queries widen many rings)"),
    "10k": dict(m=10_000, n=10_000, k=10, dist="uniform",
                workload="10K x 10K uniform, k=10 (BASELINE configs[0], the reference's serial CPU case)"),
    "100k": dict(m=100_000, n=100_000, k=10, dist="uniform",
                 workload="100K x 100K uniform, k=10 (BASELINE configs[1])"),
    "paper": dict(m=1_024_000, n=1_024_000, k=10, dist="uniform",
                  workload="1000K x 1000K uniform (the paper's rung, 1K = 1024; SURVEY §8d), k=10"),
    "dem": dict(m=4_000_000, n=4096 * 4096, k=15, dist="lattice",
                workload="4M planar data x 4096^2 raster lattice, k=15 (BASELINE configs[4])"),
}
LATTICE = 4096


def config_dict(cfg, world, scaling):
    """The `config` object — identical in both arms for the same workload."""
    n_total = cfg["n"] if scaling == "strong" else cfg["n"] * world
    return {"workload": cfg["workload"], "m": cfg["m"], "n": n_total, "k": cfg["k"],
            "distribution": cfg["dist"], "queries": f"sharded over {world} rank(s), {scaling} scaling",
            "l2": "inputs > L2 (126 MB) and L2 flushed between timed steps (256 MiB write)"}


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        p.update(hbm_gbs=float(j.get("hbm_gbs", p["hbm_gbs"])),
                 sm_max_mhz=float(j.get("sm_max_mhz", p["sm_max_mhz"])), source="measured")
        if "bf16_tflops" in j:
            p["bf16_tflops"] = float(j["bf16_tflops"])
    return p


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return platform.processor() or "unknown"


def k2_pipes(name):
    """K2's pipe utilisation from the latest committed ncu capture (the
    kernel is ALU / FP64-bound in its top-k network, so its HBM fraction is
    notional; the pipes say where it stands)."""
    import glob
    for path in reversed(sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k2_pipes.json")))):
        with open(path) as f:
            j = json.load(f)
        if j.get("config", "1m") == name:
            return {k: j[k] for k in ("alu_pipe_pct", "fp64_pipe_pct", "issue_active_pct",
                                      "dram_bytes_per_launch", "source") if k in j}
    return None


def k4_traffic(name):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K4 launch from the
    latest committed `ncu --set full` capture of this config (or None)."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k4_traffic.json")))
    for path in reversed(paths):
        with open(path) as f:
            j = json.load(f)
        if j.get("config", "1m") == name:
            return j.get("dram_bytes_per_launch")
    return None


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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

    def rows(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            pass
        return rows

    def summary(self):
        rows = self.rows()
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


def lattice_rows(world, rank, scaling):
    """Lattice rows [r0, r0 + rows) of an ny-row lattice this rank owns."""
    if scaling == "strong":
        base, extra = divmod(LATTICE, world)
        r0 = rank * base + min(rank, extra)
        return LATTICE, r0, base + (1 if rank < extra else 0)
    return LATTICE * world, LATTICE * rank, LATTICE


def lattice_box(data_bbox, ny):
    """cmd_raster's lattice box (bbox of the data, cli.hpp:495); for weak
    scaling stretched north so every rank owns 4096 rows of ny."""
    x0, y0, x1, y1 = data_bbox
    return (x0, y0, x1, y0 + (y1 - y0) * (ny // LATTICE))


def make_inputs(gen, cfg, world, rank, scaling):
    """Data and this rank's queries.  `gen` provides generate_points /
    generate_queries / generate_clustered / lattice (the repo's library in
    the GPU arm, the reference's own generator + the C restatement in the
    reference arm: bit-identical outputs, tests/test_oracle.py)."""
    m, n = cfg["m"], cfg["n"]
    n_all = n if scaling == "strong" else n * world
    if cfg["dist"] == "clustered":
        data = gen.clustered(m, 42, True)
        qx, qy = gen.clustered(n_all, 43, False)
    elif cfg["dist"] == "stress":
        data = gen.clustered(m, 42, True)
        qx, qy = gen.queries(n_all, 43)
    elif cfg["dist"] == "lattice":
        data = gen.points(m, 42, 1)
        bb = (data[0].min(), data[1].min(), data[0].max(), data[1].max())
        ny, r0, rows = lattice_rows(world, rank, scaling)
        qx, qy = gen.lattice(LATTICE, ny, lattice_box(bb, ny))
        lo, hi = r0 * LATTICE, (r0 + rows) * LATTICE
        return data, (qx[lo:hi].copy(), qy[lo:hi].copy())
    else:
        data = gen.points(m, 42, 0)
        qx, qy = gen.queries(n_all, 43)
    base, extra = divmod(n_all, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return data, (qx[lo:hi].copy(), qy[lo:hi].copy())


class RefGen:
    """Reference arm inputs: the reference's own generate_random_points /
    _queries (oracle/_ref), blob data and the lattice from the C restatement."""
    def __init__(self, O):
        self.O = O

    def points(self, m, seed, rule):
        return self.O.ref_generate_points(m, UNIT, seed, rule)

    def queries(self, n, seed):
        return self.O.ref_generate_queries(n, UNIT, seed)

    def clustered(self, n, seed, values):
        return self.O.generate_clustered(n, seed=seed, with_values=values)

    def lattice(self, nx, ny, bbox):
        return self.O.raster_lattice(nx, ny, bbox)


class LibGen:
    """GPU arm inputs from the repo's library (same bits as RefGen)."""
    def __init__(self, A):
        self.A = A

    def points(self, m, seed, rule):
        d = self.A.generate_random_points(m, UNIT, seed, "planar" if rule == 1 else "uniform")
        return d.xs, d.ys, d.zs

    def queries(self, n, seed):
        q = self.A.generate_random_queries(n, UNIT, seed)
        return q.xs, q.ys

    def clustered(self, n, seed, values):
        r = self.A.generate_clustered(n, seed=seed, with_values=values)
        return (r.xs, r.ys, r.zs) if values else (r.xs, r.ys)

    def lattice(self, nx, ny, bbox):
        q = self.A.raster_lattice(nx, ny, bbox)
        return q.xs, q.ys


def lib_inputs(A, cfg):
    """One-rank inputs as the repo's PointSets (tools / studies)."""
    (dx, dy, dz), (qx, qy) = make_inputs(LibGen(A), cfg, 1, 0, "strong")
    return A.PointSet(dx, dy, dz), A.PointSet(qx, qy)


def reference_pass(O, cfg, data, queries, stride=1, workers=0):
    """One reference cli::run_pipeline over every `stride`-th query (all the
    data): returns (wall seconds, queries interpolated, stage timings ms)."""
    qx, qy = queries
    qs = slice(0, qx.size, stride)
    t = time.perf_counter()
    _, _, tm, _ = O.ref_run_pipeline(data[0], data[1], data[2], qx[qs], qy[qs], k=cfg["k"],
                                     workers=workers)
    return time.perf_counter() - t, qx[qs].size, tm


def reference_cpu(O, cfg, data, queries, target_s=12.0):
    """The GPU arm's bounded cpu_baseline: the reference's run_pipeline on a
    strided query sample sized for ~target_s, throughput measured on it."""
    if not O.ref_available():
        return None
    threads = O.ref_hardware_threads()
    n = queries[0].size
    t, ns, _ = reference_pass(O, cfg, data, queries, stride=max(1, n // 2000))
    per_q = t / max(1, ns)
    stride = max(1, int(n / max(256, target_s / max(per_q, 1e-9))))
    t, ns, tm = reference_pass(O, cfg, data, queries, stride=stride)
    return {"value": ns / t, "unit": "points/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(), "timings_ms": tm.tolist(),
            "sample": (f"reference cli::run_pipeline (oracle/_ref, -O3 x86-64-v4 AVX-512, "
                       f"workers={threads}) on all {data[0].size} data points and every "
                       f"{stride}th query ({ns} of {n}); throughput measured on the sample "
                       f"(grid build of all data included); {t:.1f} s of CPU work")}


def repo_library_mapped():
    """True if this process has the repo's CUDA library mapped (the
    reference arm must not)."""
    try:
        with open("/proc/self/maps") as f:
            return "libaidw_b200" in f.read()
    except OSError:
        return None


def run_reference_arm(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O  # never the repo's library: this arm maps oracle/_ref only
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libaidw_ref.so not built (reference not compiled)"}))
        return 0
    threads = O.ref_hardware_threads()
    scaling = args.scaling if world > 1 else "strong"
    # the whole workload (every rank's queries): rank 0 alone interpolates it
    parts = [make_inputs(RefGen(O), cfg, world, r, scaling) for r in range(world)]
    data = parts[0][0]
    queries = (np.concatenate([p[1][0] for p in parts]), np.concatenate([p[1][1] for p in parts]))
    del parts
    n = queries[0].size
    budget = float(os.environ.get("AIDW_REF_BUDGET_S", "300"))
    # warm-up: untimed passes on a 1/64 query sample (threads, page-in),
    # which also size the timed steps
    probe = []
    for _ in range(max(1, args.warmup)):
        t, ns, _ = reference_pass(O, cfg, data, queries, stride=64)
        probe.append(t / max(1, ns))
    est_full = min(probe) * n
    stride = 1
    if est_full * args.steps > budget:
        stride = int(np.ceil(est_full * args.steps / budget))
    walls, counts, tms = [], [], []
    for _ in range(args.steps):
        t, ns, tm = reference_pass(O, cfg, data, queries, stride=stride)
        walls.append(t)
        counts.append(ns)
        tms.append(tm.tolist())
    ms_per_step = 1e3 * sum(walls) / len(walls)
    value = counts[0] / (ms_per_step / 1e3)
    serial = None
    if cfg["n"] * cfg["m"] <= 10_000 * 10_000:
        # configs[0] is the reference's serial CPU case: also one workers=1 pass
        # (executor.hpp:26-35), untimed by the driver, reported beside
        t1, ns1, _ = reference_pass(O, cfg, data, queries, stride=1, workers=1)
        serial = {"value": ns1 / t1, "unit": "points/s", "cores": 1, "s_per_pass": t1}
    sample = (f"reference cli::run_pipeline (oracle/_ref, -O3 x86-64-v4 AVX-512, "
              f"workers={threads}): " +
              (f"every step a full pass over all {n} queries and {data[0].size} data points"
               if stride == 1 else
               f"every step every {stride}th query ({counts[0]} of {n}) against all "
               f"{data[0].size} data points (K full passes would exceed {budget:.0f} s); "
               f"throughput measured on that sample"))
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the reference's generate_random_points/_queries, seeds 42/43)",
            "config": config_dict(cfg, world, scaling),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads,
                             "kind": "reference", "cpu_model": cpu_model(),
                             "sampled": stride > 1, "sample": sample,
                             "stage_ms_first_step": {"build": tms[0][0], "knn": tms[0][1],
                                                     "interp": tms[0][2]}},
            **({"serial_workers1": serial} if serial else {}),
            "repo_library_mapped": repo_library_mapped(),
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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: shard configs[2]'s 1M queries (strong, default) or run 1M per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--verify", action="store_true",
                    help="check the gathered shards against one device's run of all queries")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1601_05904_b200 as A
    from paper_1601_05904_b200 import shard

    world, rank, local = dist_env()
    scaling = args.scaling if world > 1 else "strong"
    # AIDW_BENCH_SHARED_DEVICE=1 (test hook): every rank on device 0 with the
    # gloo backend, so the multi-rank path runs end to end on a one-GPU box
    shared = os.environ.get("AIDW_BENCH_SHARED_DEVICE") == "1"
    local = 0 if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # everything on one non-default stream: the L2 flush, the inputs and the
    # library's work are stream-ordered (a NULL stream handle would make the
    # library use its own stream, not ordered after the flush), and the
    # events time exactly that stream
    torch.cuda.set_stream(torch.cuda.Stream(dev))
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
        t = torch.tensor([x], dtype=torch.float64, device=dev if not shared else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    name, sms = A.device_info()
    gen = LibGen(A)
    lattice = cfg["dist"] == "lattice"

    class Job:
        """One workload shard resident in HBM (data replicated by broadcast)."""
        def __init__(self, sc):
            self.sc = sc
            (dxs, dys, dzs), (qxs, qys) = make_inputs(gen, cfg, world, rank, sc)
            self.host = (dxs, dys, dzs, qxs, qys)
            self.m, self.n = dxs.size, qxs.size
            self.n_total = cfg["n"] if sc == "strong" else cfg["n"] * world
            self.d_data = torch.from_numpy(np.stack([dxs, dys, dzs])).to(dev)
            if world > 1:
                if shared:
                    cpu = self.d_data.cpu()
                    shard.replicate(cpu, dist)
                    self.d_data.copy_(cpu)
                else:
                    shard.replicate(self.d_data, dist)
            self.d_q = torch.from_numpy(np.stack([qxs, qys])).to(dev)
            self.d_pred = torch.empty(self.n, dtype=torch.float64, device=dev)
            self.d_alpha = torch.empty(self.n, dtype=torch.float64, device=dev)
            self.stream = torch.cuda.current_stream(dev)
            self.sp = self.stream.cuda_stream
            self.dx, self.dy, self.dz = (self.d_data[i].data_ptr() for i in range(3))
            self.qx, self.qy = self.d_q[0].data_ptr(), self.d_q[1].data_ptr()
            if lattice:
                dbb = A.compute_bbox_device(self.dx, self.dy, self.m, self.qx, self.qy, 0, self.sp)
                self.ny, self.r0, self.rows = lattice_rows(world, rank, sc)
                self.lbox = lattice_box(tuple(dbb), self.ny)
            # global bbox(data ∪ all queries): per-rank device reduce + all-reduce
            bb = A.compute_bbox_device(self.dx, self.dy, self.m, self.qx, self.qy, self.n, self.sp)
            bb = shard.global_bbox(bb, dist if world > 1 else None,
                                   device=dev if not shared else None)
            self.rc = A.RunConfig(params=A.AidwParams(k=cfg["k"]), bbox=tuple(float(v) for v in bb))
            self.rc_c = self.rc.c()
            self.pp, self.pa = self.d_pred.data_ptr(), self.d_alpha.data_ptr()

        def step(self):
            """One pass; returns the raw C stats (converted after timing)."""
            if lattice:  # cmd_raster: this rank's lattice rows generated in HBM each step
                A.raster_lattice_device(LATTICE, self.ny, self.lbox, self.qx, self.qy, self.r0,
                                        self.rows, self.sp)
            return A.run_pipeline_device(self.dx, self.dy, self.dz, self.m, self.qx, self.qy,
                                         self.n, self.rc_c, self.pp, self.pa, self.sp, raw=True)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def timed(job, steps, warmup, clocks=None):
        for _ in range(warmup):
            flush.zero_()
            job.step()
        barrier()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        stats = []
        l0 = A.kernel_launch_count()
        barrier()
        for i in range(steps):
            flush.zero_()  # L2 flush between timed steps (256 MiB write), not timed
            starts[i].record(job.stream)
            stats.append(job.step())
            ends[i].record(job.stream)
        barrier()
        launches = A.kernel_launch_count() - l0
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        return allmax(sum(step_ms)) / steps, [st.as_dict() for st in stats], launches

    job = Job(scaling)
    m, n = job.m, job.n
    with ClockSampler(local) as clocks:
        time.sleep(0.2)
        ms_per_step, stats, launches = timed(job, args.steps, args.warmup)
        # short workloads (10K): keep stepping, untimed, until the sampler has
        # seen the GPU under this load a few times
        t_end = time.time() + 2.0
        while len(clocks.rows()) < 6 and time.time() < t_end:
            job.step()
            torch.cuda.synchronize()
    value = job.n_total / (ms_per_step / 1e3)

    # roofline of the dominant kernel (K4): live CUDA-event duration of the
    # weight_fp32_kernel launch inside each timed step (this rank's shard)
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
    engine = A.weight_engine(m)  # a function of m: "tensor-core" or "cuda-core"
    tc = engine == "tensor-core"
    # Pipe roofline of the executed formula mix (K4 far-tile forms):
    # per SM and clock the FMA pipe retires 128 FP32 ops (FFMA2 = 2, measured
    # profiles/r02/tmem_bench.txt) and the XU pipe 16 MUFU ops; a class is
    # bound by the slower of the two.
    #   recipe (alpha == 4), CUDA-core engine: 3 (d2) + 1 (d2^2) + 2.5 (pair /
    #     single sums) = 6.5 FP32 + 0.75 MUFU per pair
    #   recipe, tensor-core engine: d2 from the tcgen05 MMA; 1 (d2^2) + 3
    #     (two points per reciprocal) = 4 FP32 + 0.5 MUFU per pair — both pipes
    #     at 32 pairs / SM-clk
    #   general (CUDA-core engine in both): G1 6 FP32 + 2 MUFU (lg2, ex2), G2
    #     14 FP32 + 1 MUFU (ex2 as a degree-5 polynomial); G1 / G2 split ~1:1
    ops_recipe = 4.0 if tc else 6.5
    clk_recipe = max(4.0 / 128, 0.5 / 16) if tc else max(6.5 / 128, 0.75 / 16)
    clk_general = max(0.5 * (6 + 14) / 128, 0.5 * (2 + 1) / 16)
    clk_mix = (a4 * clk_recipe + (n - a4) * clk_general) / n
    peak_mix = sms * f_mhz * 1e6 / clk_mix / 1e9
    peak_general = sms * f_mhz * 1e6 / clk_general / 1e9
    ops_mix = (a4 * ops_recipe + (n - a4) * 10.0) / n
    k4_kernel = ("weight_tc_kernel (K4 recipe queries: tcgen05 kind::tf32 d2 into TMEM) + "
                 "weight_fp32_kernel (general-alpha queries, side stream)" if tc
                 else "weight_fp32_kernel (K4)")
    recipe_form = ("tensor-core engine: d2 by MMA, 4 FP32 + 0.5 MUFU" if tc
                   else "FMA-bound 6.5 FP32 + 0.75 MUFU")

    # general-alpha path forced (every query on exp2/log2), reported separately
    A.set_alpha4_recipe(False)
    gen_stats = []
    for _ in range(2):
        flush.zero_()
        gen_stats.append(job.step().as_dict())
    A.set_alpha4_recipe(True)
    k4g_ms = statistics.median(s["weight_kernel_ms"] for s in gen_stats)
    torch.cuda.synchronize()

    # the reference's precision: FP64 weighting kernel, same pipeline
    fp64 = None
    if not args.no_fp64:
        A.set_weight_precision("fp64")
        ms64, st64, _ = timed(job, 2, 1)
        A.set_weight_precision("fp32")
        fp64 = {"value": job.n_total / (ms64 / 1e3), "unit": "points/s", "ms_per_step": ms64,
                "k4_ms": statistics.median(s["weight_kernel_ms"] for s in st64),
                "kernel": "weight_fp64_kernel<BLOCKED> (AIDW_WEIGHT_FP64=1)"}

    # --verify: the ranks' shards, gathered, equal one device's run of the
    # whole query set bit for bit (the invariance the sharding relies on)
    verify = None
    if args.verify and scaling == "strong":
        job.step()
        torch.cuda.synchronize()
        mine = torch.stack([job.d_pred, job.d_alpha]).cpu()
        if world > 1:
            parts = [None] * world
            dist.all_gather_object(parts, mine)
        else:
            parts = [mine]
        if rank == 0:
            got = torch.cat(parts, dim=1)
            (dxs_, dys_, dzs_), (qxs_, qys_) = make_inputs(gen, cfg, 1, 0, "strong")
            d_all = torch.from_numpy(np.stack([dxs_, dys_, dzs_])).to(dev)
            q_all = torch.from_numpy(np.stack([qxs_, qys_])).to(dev)
            p_all = torch.empty(qxs_.size, dtype=torch.float64, device=dev)
            a_all = torch.empty(qxs_.size, dtype=torch.float64, device=dev)
            if lattice:
                A.raster_lattice_device(LATTICE, LATTICE, job.lbox, q_all[0].data_ptr(),
                                        q_all[1].data_ptr(), 0, LATTICE, job.sp)
            A.run_pipeline_device(d_all[0].data_ptr(), d_all[1].data_ptr(), d_all[2].data_ptr(),
                                  dxs_.size, q_all[0].data_ptr(), q_all[1].data_ptr(), qxs_.size,
                                  job.rc, p_all.data_ptr(), a_all.data_ptr(), job.sp)
            torch.cuda.synchronize()
            ref = torch.stack([p_all, a_all]).cpu()
            verify = {"shards_bit_identical": bool(torch.equal(got, ref)), "n": int(got.shape[1])}
        if world > 1:
            dist.barrier()

    # weak-scaling figure beside the strong one (N > 1): 1M queries per rank
    weak = None
    if world > 1 and scaling == "strong":
        wjob = Job("weak")
        wms, _, _ = timed(wjob, min(args.steps, 3), 1)
        weak = {"value": wjob.n_total / (wms / 1e3), "unit": "points/s", "ms_per_step": wms,
                "n": wjob.n_total, "per_rank": wjob.n}
        del wjob

    # e2e through the public C-ABI with pinned host buffers
    dxs, dys, dzs, qxs, qys = job.host
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in
           dict(dx=dxs, dy=dys, dz=dzs, qx=qxs, qy=qys).items()}
    hd = A.PointSet(pin["dx"].numpy(), pin["dy"].numpy(), pin["dz"].numpy())
    hq = A.PointSet(pin["qx"].numpy(), pin["qy"].numpy())
    hcfg = A.RunConfig(params=A.AidwParams(k=cfg["k"]), bbox=job.rc.bbox)
    raster_e2e = lattice and world == 1
    if raster_e2e:
        # the public raster call: host data in, raster out (lattice in HBM)
        rcfg = A.RunConfig(params=A.AidwParams(k=cfg["k"]))

        def e2e_call():
            return A.run_raster(hd, LATTICE, LATTICE, rcfg, with_alpha=False)
    else:
        # results land in pinned host buffers (the C-ABI writes caller memory)
        pout = (torch.empty(n, dtype=torch.float64).pin_memory().numpy(),
                torch.empty(n, dtype=torch.float64).pin_memory().numpy())

        def e2e_call():
            return A.run_pipeline(hd, hq, hcfg, out=pout)
    e2e_call()
    barrier()
    # at least --e2e-steps calls and ~0.3 s of them (small configs: host-clock noise)
    e2e_steps = max(args.e2e_steps, int(np.ceil(0.3 / max(ms_per_step / 1e3, 1e-6))))
    e2e_steps = int(allmax(e2e_steps))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    barrier()
    e2e_s = allmax((time.perf_counter() - t0) / e2e_steps)
    e2e_value = job.n_total / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O  # checker / baseline only, outside every timed region
        cpu = reference_cpu(O, cfg, (dxs, dys, dzs), (qxs, qys))
        if cpu is None:
            cpu = {"value": None, "unit": "points/s", "cores": 0, "kind": "reference",
                   "sample": "oracle/_ref not available"}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32 weighting / f64 grid+kNN+alpha",
            "data": "synthetic (the reference's mt19937_64 generators, seeds 42/43)",
            "config": config_dict(cfg, world, scaling),
            "hardware": {"device": name, "sms": sms, "per_rank_queries": n,
                         "data_replication": "NCCL broadcast from rank 0" if world > 1 else "none"},
            "roofline": {"bound": "fp32+mufu pipes", "kernel": k4_kernel, "engine": engine,
                         "achieved": achieved, "peak": peak_mix, "unit": "Gpair/s",
                         "frac": achieved / peak_mix, "traffic": k4_traffic(args.config),
                         "peak_def": f"{sms} SMs x {f_mhz:.0f} MHz ({pk['source']} sm_max_mhz) / "
                                     f"{clk_mix:.4f} SM-clk per pair: executed mix of the "
                                     f"alpha=4 recipe ({a4} queries; {recipe_form}) and "
                                     f"general alpha (MUFU-bound 10 FP32 + 1.5 MUFU) far-tile "
                                     f"forms; 128 FP32 + 16 MUFU per SM-clk",
                         "frac_vs_2mufu_roofline": achieved / peak_gpairs,
                         "fp32_view": {  # the same bound as FP32 op throughput
                             "unit": "TFLOP/s (FP32 ops, FFMA = 1)",
                             "ops_per_pair": ops_mix,
                             "achieved": achieved * 1e9 * ops_mix / 1e12,
                             "peak": sms * 128 * f_mhz * 1e6 / 1e12,
                             "frac": achieved * 1e9 * ops_mix / (sms * 128 * f_mhz * 1e6)},
                         "alpha4_recipe_queries": a4, "pairs_per_launch": pairs,
                         "k4_ms": k4_ms},
            # the tensor-core share of K4 (recipe queries): kind::tf32 MMA,
            # K = 16 (exact TF32 pieces) -> 32 flops per pair; dense TF32 peak
            # taken as half the measured bf16 figure
            "tensor_view": ({"mma": "tcgen05.mma.cta_group::1.kind::tf32 M128 N64 K16 (2 x K8)",
                             "flops_per_pair": 32,
                             "achieved_tflops": a4 * m * 32 / (k4_ms / 1e3) / 1e12,
                             "peak_tflops": pk.get("bf16_tflops", 2250.0) / 2,
                             "frac": a4 * m * 32 / (k4_ms / 1e3) / 1e12 /
                                     (pk.get("bf16_tflops", 2250.0) / 2)} if tc else None),
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
                            "candidates_reference": ref_cand, "candidates_scanned": cand,
                            "pipes_ncu": k2_pipes(args.config),
                            "note": "algorithmic bytes credit the reference's candidates; "
                                    "the kernel is ALU/FP64-bound in its top-k network "
                                    "(profiles/r02)"},
                "build_hbm": {"bytes": build_bytes,
                              "achieved_gbs": build_bytes / (build_ms / 1e3) / 1e9,
                              "frac": build_bytes / (build_ms / 1e3) / 1e9 / pk["hbm_gbs"]},
                "weight_ms": k4_ms, "interp_ms": statistics.median(s["interp_ms"] for s in stats),
            },
            "e2e": {"value": e2e_value, "unit": "points/s",
                    "api": "aidw_run_raster (C-ABI)" if raster_e2e else "aidw_run_pipeline (C-ABI)",
                    "h2d_bytes_per_step": 24 * m + (0 if raster_e2e else 16 * n),
                    "d2h_bytes_per_step": (8 if raster_e2e else 16) * n,
                    "s_per_step": e2e_s, "calls": e2e_steps},
            "gpu_launches": launches,
            "cuda_graphs": A.graph_counters(),
            "clocks": clk,
        }
        if fp64 is not None:
            line["fp64"] = fp64
        if weak is not None:
            line["weak_scaling"] = weak
        if verify is not None:
            line["verify"] = verify
        if cpu is not None:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")
                                    if k in cpu}
            line["cpu_baseline"]["cpu_model"] = cpu.get("cpu_model", cpu_model())
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
