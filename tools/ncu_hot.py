"""Summarise an ncu --page source --csv --print-source sass export: per-SASS
instruction stall samples, grouped into regions between labelled anchors.

    ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_hot.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, h):
    try:
        return float(r[col[h]] or 0)
    except ValueError:
        return 0.0


tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total samples {tot:.0f}")
agg = {h: sum(num(r, h) for r in data) for h in reasons}
print("by reason:", ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for h, v in
                               sorted(agg.items(), key=lambda x: -x[1]) if v / tot > 0.005))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hot = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]
for r in hot:
    s = num(r, "Warp Stall Sampling (All Samples)")
    why = sorted(((num(r, h), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{r[col['Address']]:>6} {100 * s / tot:5.2f}%  {r[col['Source']][:70]:70s} "
          + " ".join(f"{n}:{100 * v / tot:.2f}" for v, n in why if v))
