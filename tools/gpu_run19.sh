PDQ_LIB=tools/libvar_def1.so timeout 300 python tools/leaf_check.py 2>&1 | tail -1
for v in def0 def1 def0 def1; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 5 2>&1 | tail -2; done
PDQ_LIB=tools/libvar_def1.so timeout 300 python tools/small_n.py 2>&1 | grep '"depth_limit": 0'
