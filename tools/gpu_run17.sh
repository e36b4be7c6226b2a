timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/prof_sort.py 28 i32 2 1,2,3,4,6,8,9,10,11,12,13,14,15,16 2>&1 | tail -15
