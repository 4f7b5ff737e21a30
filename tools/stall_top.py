"""Top stalled instructions of an `ncu --page source --csv` export, with the
three largest stall reasons of each and a per-reason total (development aid).
usage: python tools/stall_top.py <source.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_")]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r[1], float(r[ix["Warp Stall Sampling (All Samples)"]]),
                     float(r[ix["Instructions Executed"]]), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data)
print("total samples", tot, "instructions", len(data))
agg = {k: 0.0 for k in reasons}
for d in data:
    for k in reasons:
        v = d[4][ix[k]]
        if v not in ("", "0"):
            agg[k] += float(v)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                              sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0.005 * tot))
for a, s, sm, ie, r in sorted(data, key=lambda d: -d[2])[:top_n]:
    st = {k: float(r[ix[k]]) for k in reasons if r[ix[k]] not in ("", "0")}
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{a:#x} {100 * sm / tot:5.2f}% exec={ie:.3g} {s[:58]:58s}",
          " ".join(f"{k[6:]}:{v:.0f}" for k, v in big))
