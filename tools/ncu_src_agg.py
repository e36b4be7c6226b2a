"""Aggregate an ncu --page source --csv --print-source cuda,sass export by (file, line): warp-stall
samples and executed instructions; prints the top lines with their source text.
  python tools/ncu_src_agg.py report_source.csv [top] [src_root]"""
import collections
import csv
import os
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
root = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "paper_2106_05123_b200", "csrc")
rows = list(csv.reader(open(path)))
hdr, fname = None, None
samp, inst = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(d["Line No"])
    except ValueError:
        continue
    samp[(fname, ln)] += float((d.get("Warp Stall Sampling (All Samples)") or "0").replace(",", ""))
    inst[(fname, ln)] += float((d.get("Instructions Executed") or "0").replace(",", ""))
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
cache = {}


def text(f, ln):
    p = os.path.join(root, f)
    if p not in cache:
        cache[p] = open(p).read().split("\n") if os.path.exists(p) else []
    lines = cache[p]
    return lines[ln - 1].strip()[:100] if 0 < ln <= len(lines) else ""


print(f"samples {ts:.0f} instructions {ti:.3g}")
for (f, ln), v in samp.most_common(top):
    print(f"{v / ts:.3f} {inst[(f, ln)] / ti:.3f} {f}:{ln}: {text(f, ln)}")
