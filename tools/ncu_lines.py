"""Aggregate an ncu source page (cuda,sass) by source line: samples, stall reasons, instructions.

usage: python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
SORTKEY = "Instructions Executed" if "--by-inst" in sys.argv else "Warp Stall Sampling (All Samples)"
sys.argv = [a for a in sys.argv if a != "--by-inst"]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: defaultdict(int))
src_text = {}
hdr = None
cur_file = None
cur_line = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0]:  # a source line row
        cur_line = (cur_file, int(r[0]))
        src_text[cur_line] = r[1].strip()[:70]
        continue
    if cur_line is None:
        continue
    d = agg[cur_line]
    for i, h in enumerate(hdr):
        if i < 4 or i >= len(r):
            continue
        if h in ("Warp Stall Sampling (All Samples)", "Instructions Executed") or (h.startswith("stall_") and "Not Issued" not in h):
            try:
                d[h] += int(r[i] or 0)
            except ValueError:
                pass
tot_s = sum(d["Warp Stall Sampling (All Samples)"] for d in agg.values()) or 1
tot_i = sum(d["Instructions Executed"] for d in agg.values()) or 1
print(f"total samples {tot_s}  warp-instructions {tot_i:.3g}")
for key, d in sorted(agg.items(), key=lambda kv: -kv[1][SORTKEY])[:top]:
    st = sorted(((v, k[6:]) for k, v in d.items() if k.startswith("stall_")), reverse=True)[:3]
    sts = " ".join(f"{k}:{v / max(1, d['Warp Stall Sampling (All Samples)']):.2f}" for v, k in st if v)
    print(f"{d['Warp Stall Sampling (All Samples)'] / tot_s:6.3f} inst {d['Instructions Executed'] / tot_i:6.3f} "
          f"{key[0]}:{key[1]:<5d} {src_text.get(key, ''):70s} {sts}")
