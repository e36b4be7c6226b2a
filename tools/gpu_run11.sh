PDQ_LIB=tools/libvar_sp2.so timeout 300 python tools/leaf_check.py 2>&1 | tail -1
PDQ_LIB=tools/libvar_sp2.so timeout 300 python tools/small_n.py 2>&1 | grep '"depth_limit": 0'
for v in wn3 sp2; do PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 4 2>&1 | tail -1; done
