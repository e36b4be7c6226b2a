timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/leaf_check.py 2>&1 | tail -1
timeout 600 python tools/fallback_bench.py 28 2>&1 | grep -v k16
timeout 600 python tools/fallback_bench.py 24 2>&1 | head -2
timeout 300 python tools/small_n.py 2>&1 | grep '"depth_limit": 0'
timeout 900 python bench.py > gpurun_out/bench_R14.json 2> gpurun_out/bench_R14.err; tail -2 gpurun_out/bench_R14.err
