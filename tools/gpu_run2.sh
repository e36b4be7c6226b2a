set -x
PDQ_LIB=tools/libvar_wnet.so timeout 300 python tools/leaf_check.py 2>&1 | tail -5
for v in old wnet; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 4 2>&1 | tail -2; done
timeout 600 python tools/host_probe.py 2>&1 | tail -16
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
