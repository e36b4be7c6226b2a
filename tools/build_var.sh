#!/bin/bash
# Profiling variant: int32 keys-only library at tools/libvar_<name>.so with extra -D flags.
#   tools/build_var.sh <name> [-DPDQ_X=..]...   then run with PDQ_LIB=tools/libvar_<name>.so
cd "$(dirname "$0")/.." || exit 1
name=$1; shift
python - "$name" "$@" > /tmp/build_$name.log 2>&1 <<'PY'
import sys
from paper_2106_05123_b200 import _lib
name, extra = sys.argv[1], sys.argv[2:]
_lib.build(verbose=True, out=f"tools/libvar_{name}.so", extra_flags=extra, only_i32=True)
PY
rc=$?; echo "build $name rc=$rc"; grep -E "error" /tmp/build_$name.log | head
grep -A1 -E "Compiling entry function '_ZN3pdq6k_(sort|base)IjLb0ELb0" /tmp/build_$name.log | grep -o "Used.*"
cuobjdump -sass tools/libvar_$name.so > /tmp/var_$name.sass
python3 - "$name" <<'PY'
import re,sys
s=open(f'/tmp/var_{sys.argv[1]}.sass').read()
for p in s.split("Function : ")[1:]:
    name=p.split("\n",1)[0]
    print(name[:40], "LDL/STL", len(re.findall(r"\b(LDL|STL)", p)))
PY
exit $rc
