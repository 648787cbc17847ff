"""Write profiles/<round>/k4_traffic.json from an `ncu --set full` capture of
the dominant K4 kernel (dram__bytes_read.sum + dram__bytes_write.sum per
launch), which bench.py reports as roofline.traffic.

    python tools/k4_traffic.py gpurun_out/k4tc_r02.ncu-rep profiles/r02/k4_traffic.json \
        --kernel weight_tc_kernel --config 1m
"""
import argparse
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("out")
ap.add_argument("--kernel", default="weight_tc_kernel")
ap.add_argument("--config", default="1m")
args = ap.parse_args()
raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    rec = dict(zip(hdr, r))
    if args.kernel not in rec.get("Kernel Name", ""):
        continue
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = {}
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u = units[hdr.index(key)]
        vals[key] = float(rec[key].replace(",", "")) * scale.get(u, 1)
    out = {"kernel": args.kernel, "config": args.config,
           "dram_bytes_read": int(vals["dram__bytes_read.sum"]),
           "dram_bytes_write": int(vals["dram__bytes_write.sum"]),
           "dram_bytes_per_launch": int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]),
           "source": f"ncu --set full --clock-control none ({args.rep.split('/')[-1]})"}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))
    break
else:
    raise SystemExit(f"{args.kernel} not in {args.rep}")
