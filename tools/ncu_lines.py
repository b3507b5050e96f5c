"""Aggregate ncu source-page stall samples per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME --launch-count 1 > x.csv
       python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
cur_file, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    agg.setdefault(key, [0.0, r[1]])
    agg[key][0] += v
tot = sum(v for v, _ in agg.values()) or 1
for (f, ln), (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v / tot:6.1%} {f}:{ln}: {src.strip()[:100]}")
