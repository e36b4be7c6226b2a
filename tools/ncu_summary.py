"""Summarise ncu --set full reports per kernel (duration, DRAM bytes, occupancy, issue) into JSON.

python tools/ncu_summary.py out.json report1.ncu-rep [report2.ncu-rep ...]
bench.py reads the newest profiles/r*_ncu_kernels.json for roofline.traffic.
"""
import csv
import io
import json
import re
import subprocess
import sys

FIELDS = {
    "gpu__time_duration.sum": ("duration_ms", {"ms": 1, "us": 1e-3, "ns": 1e-6}),
    "dram__bytes_read.sum": ("dram_read_GB", {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}),
    "dram__bytes_write.sum": ("dram_write_GB", {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}),
    "launch__registers_per_thread": ("registers", None),
    "launch__grid_size": ("grid", None),
    "launch__block_size": ("block", None),
    "sm__inst_issued.avg.pct_of_peak_sustained_active": ("issue_active_pct", None),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("warps_active_pct", None),
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("dram_throughput_pct", None),
    "lts__t_sector_hit_rate.pct": ("l2_hit_pct", None),
}

out = {}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        name = re.sub(r"<.*", "", row[hdr.index("Kernel Name")].replace("void ", "")).split("(")[0].strip()
        name = name.split("::")[-1]
        d = {"report": rep.split("/")[-1]}
        for metric, (key, scale) in FIELDS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                if scale:
                    v *= scale.get(units[i], 1)
                d[key] = v
        out.setdefault(name, d)  # first launch of each kernel
with open(sys.argv[1], "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
