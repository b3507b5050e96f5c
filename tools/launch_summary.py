"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
usage: python tools/launch_summary.py launches.csv [header line]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
agg = {}
for r in rows:
    if r[12] != "gpu__time_duration.sum":
        continue
    name = r[4].split("(")[0].replace("kkt::", "").replace("void ", "")
    ns = float(r[14].replace(",", "")) * (1e3 if r[13] == "us" else 1e6 if r[13] == "ms" else 1)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ns
tot = sum(v[1] for v in agg.values()) or 1
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {c:8d} {ns / 1e6:10.3f} {ns / tot:7.1%}")
