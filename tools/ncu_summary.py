"""Summarise ncu captures into profiles/<round>/ (markdown).

    python tools/ncu_summary.py gpurun_out/k4_r01.ncu-rep [...] --launches gpurun_out/launches_r01.csv \
        --out profiles/r01/ncu_summary.md
"""
import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active", "TMA pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid size"),
    ("launch__block_size", "block size"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    h, u, data = raw(rep)
    lines = [f"### `{rep.split('/')[-1]}`", ""]
    for row in data:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines += [f"kernel: `{name[:120]}`", "", "| metric | value | unit |", "|---|---|---|"]
        for k, label in KEYS:
            if k in h:
                lines.append(f"| {label} (`{k}`) | {row[h.index(k)]} | {u[h.index(k)]} |")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and k.endswith(("_not_issued",)) is False:
                try:
                    stalls.append((float(row[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            tot = sum(v for v, _ in stalls) or 1.0
            lines += ["", "top stall reasons (pc sampling): " +
                      ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in stalls[:6])]
        lines.append("")
    return lines


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], float(d["Metric Value"]), d["Metric Unit"]))
    tot = sum(v for _, v, _ in out) or 1.0
    lines = ["### launch list (one fused pipeline pass, `gpu__time_duration.sum`, "
             "--clock-control none; cold-cache, serialised: compare shares)", "",
             "| kernel | time | share |", "|---|---|---|"]
    agg = {}
    for n, v, unit in out:
        key = n.split("(")[0].replace("(anonymous namespace)::", "")[:70]
        agg.setdefault(key, [0.0, 0, unit])
        agg[key][0] += v
        agg[key][1] += 1
    for k, (v, c, unit) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"| `{k}` x{c} | {v:,.0f} {unit} | {100 * v / tot:.2f}% |")
    lines.append(f"| total ({len(out)} launches) | {tot:,.0f} | 100% |")
    return lines + [""]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        lines += launches(a.launches)
    for r in a.reports:
        lines += summarise(r)
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
