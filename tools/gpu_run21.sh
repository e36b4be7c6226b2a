PDQ_LIB=tools/libvar_ring.so timeout 300 python tools/leaf_check.py 2>&1 | tail -1
for v in rev ring rev ring; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 300 python tools/small_n.py 2>&1 | grep '"depth_limit": 0' | head -3; done
