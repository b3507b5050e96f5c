"""Summarise an ncu --set full report: per kernel duration, DRAM traffic, occupancy, top
warp-stall reasons.  usage: python tools/ncu_summary.py report.ncu-rep > profiles/x.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def g(r, k):
    i = col.get(k)
    return (r[i], units[i]) if i is not None else ("n/a", "")


print(f"ncu --set full summary of {rep.split('/')[-1]}\n")
for r in rows[2:]:
    name = r[col["Kernel Name"]][:70]
    dur, du = g(r, "gpu__time_duration.sum")
    rd, ru = g(r, "dram__bytes_read.sum")
    wr, wu = g(r, "dram__bytes_write.sum")
    occ, _ = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    iss, _ = g(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    dram, _ = g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    regs, _ = g(r, "launch__registers_per_thread")
    grid, _ = g(r, "launch__grid_size")
    blk, _ = g(r, "launch__block_size")
    print(f"{name}\n  time {dur} {du}; DRAM read {rd} {ru}, write {wr} {wu}; DRAM thrpt {dram}% of peak")
    print(f"  grid {grid} x block {blk}, regs {regs}; warps active {occ}% ; issue active {iss}%")
    st = []
    for h, i in col.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]) + "\n")
