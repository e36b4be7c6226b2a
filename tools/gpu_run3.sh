set -x
PDQ_LIB=tools/libvar_wnet.so timeout 300 python tools/leaf_check.py 2>&1 | tail -5
for v in old wnet; do echo "== $v"; PDQ_LIB=tools/libvar_$v.so timeout 120 python tools/prof_sort.py 28 i32 4 2>&1 | tail -2; done
timeout 600 python tools/host_probe.py 2>&1 | grep chunk_kb | grep -v host_register
timeout 600 python bench.py --no-cpu > gpurun_out/bench_R3.json 2>gpurun_out/bench_R3.err; tail -2 gpurun_out/bench_R3.err
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_C1.json 2>&1
