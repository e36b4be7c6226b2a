PDQ_LIB=tools/libvar_pdl.so timeout 300 python tools/leaf_check.py 2>&1 | tail -1
PDQ_LIB=tools/libvar_pdl.so timeout 300 python tools/small_n.py 2>&1 | grep '"depth_limit": 0'
PDQ_LIB=tools/libvar_pdl.so timeout 120 python tools/prof_sort.py 28 i32 5 2>&1 | tail -2
PDQ_LIB=tools/libvar_pdl.so timeout 120 python tools/fallback_bench.py 24 2>&1 | head -2
