#!/bin/bash
# Build libpdq_b200.so with -Xptxas -v and summarise registers / local-memory use of k_sort.
cd "$(dirname "$0")/.." || exit 1
python -c "from paper_2106_05123_b200 import _lib; _lib.build(verbose=True, extra_flags=['-DPDQ_BUILD_CHECK'])" > /tmp/build.log 2>&1
rc=$?; echo "build rc=$rc"; grep -E "error" /tmp/build.log | head
awk '/Compiling entry function/{name=$0} /Used [0-9]+ registers/{print name " :: " $0}' /tmp/build.log | sed 's/ptxas info    ://g; s/Compiling entry function//' | grep k_sort | cut -c1-160
cuobjdump -sass paper_2106_05123_b200/libpdq_b200.so > /tmp/all.sass
python3 - <<'PY'
import re
s=open('/tmp/all.sass').read()
for p in s.split("Function : "):
    name=p.split("\n",1)[0]
    if "k_sort" in name:
        print(name[:40], "lines", len(p.split("\n")), "LDL/STL", len(re.findall(r"\b(LDL|STL)", p)), "UBLKCP", len(re.findall("UBLKCP", p)))
PY
exit $rc
