"""Per-kernel DRAM bytes from an ncu --set full report (first launch of each kernel) ->
profiles/<round>_ncu_traffic.json, read by bench.py for the roofline's `traffic` field.
usage: python tools/ncu_traffic.py report.ncu-rep out.json"""
import csv
import io
import json
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "msecond": 1.0,
         "usecond": 1e-3, "nsecond": 1e-6}


def val(r, k):
    i = col[k]
    return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)


kern = {}
for r in rows[2:]:
    name = re.sub(r"\(DevPlan.*$|\(kkt::DevPlan.*$", "", r[col["Kernel Name"]])
    name = re.sub(r"^void ", "", name).replace("kkt::", "").replace("(int)", "")
    if name in kern:
        continue
    kern[name] = {"dram_read_bytes": val(r, "dram__bytes_read.sum"),
                  "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                  "duration_ms": val(r, "gpu__time_duration.sum")}
json.dump({"source": f"ncu --set full --clock-control none ({rep.split('/')[-1]}), B=64, first launch of each kernel",
           "kernels": kern}, open(out, "w"), indent=1)
print(json.dumps(kern, indent=1))
