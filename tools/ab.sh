for v in "$@"; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 4 "" x 2>&1 | tail -3; done
