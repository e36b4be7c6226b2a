for v in base32 c16 c32d4 base32 c16 c32d4; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 5 2>&1 | tail -2; done
PDQ_LIB=tools/libvar_c16.so timeout 600 python tools/prof_sort.py 28 i32 2 1,2,11,12 2>&1 | tail -4
