timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fallback or bad_shift" 2>&1 | tail -2
timeout 600 python tools/fallback_bench.py 28 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
