"""SASS opcode histogram per kernel of the built library (static instruction counts), highlighting the
instructions that show the Blackwell features in use (UBLKCP = TMA bulk copy, SYNCS = mbarrier,
griddepcontrol = ACQBULK/...), for profiles/.
  python tools/sass_hist.py [lib.so] > profiles/r02_sass_histogram.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2106_05123_b200/libpdq_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
want = {"k_sort": r"_ZN3pdq6k_sortIjLb0ELb0EEEvNS_6ParamsE", "k_base_big": r"_ZN3pdq10k_base_bigILb0EEEvNS_6ParamsE",
        "k_base_wide (int64,u32)": r"_ZN3pdq11k_base_wideImLb0ELb1EEEvNS_6ParamsE",
        "k_check": r"_ZN3pdq7k_checkIjLb0ELb0EEEvNS_6ParamsE", "k_init": r"_ZN3pdq6k_initIjLb0ELb0EEEvNS_6ParamsE"}
print(f"# static SASS opcode counts per kernel ({lib}; cuobjdump -sass); int32 keys-only instantiations unless noted")
for label, mangled in want.items():
    body = next((f for f in funcs if f.startswith(mangled)), None)
    if body is None:
        print(f"\n## {label}: not found")
        continue
    ops = collections.Counter()
    for line in body.split("\n"):
        m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            ops[m.group(1)] += 1
    total = sum(ops.values())
    print(f"\n## {label}: {total} instructions")
    feat = {k: ops.get(k, 0) for k in ("UBLKCP", "SYNCS", "UTMALDG", "VOTE", "REDUX", "MATCH", "ATOMS", "ATOMG", "RED",
                                         "BAR", "SHFL", "VIMNMX", "VIMNMX3", "LDS", "STS", "LDG", "STG", "LDL", "STL",
                                         "ACQBULK", "CCTL")}
    print("features: " + ", ".join(f"{k} {v}" for k, v in feat.items() if v))
    print("top: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(25)))
