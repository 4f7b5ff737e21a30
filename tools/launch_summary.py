"""Per-kernel share of GPU time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).
usage: python tools/launch_summary.py X.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ui = h.index("Metric Unit")
scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3,
         "s": 1.0, "second": 1.0, "nsecond": 1e-9}
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-9)
    cnt[name] += 1
all_t = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'seconds':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.4f} {100 * v / all_t:6.2f}%")
print(f"{'total':60s} {sum(cnt.values()):8d} {all_t:10.4f}")
