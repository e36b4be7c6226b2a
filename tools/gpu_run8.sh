PDQ_LIB=tools/libvar_wn2.so timeout 300 python tools/leaf_check.py 2>&1 | tail -2
for v in wnet wn2; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 4 2>&1 | tail -2; done
