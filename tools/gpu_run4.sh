set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fallback or bad_shift" 2>&1 | tail -5
timeout 600 python tools/fallback_bench.py 28 2>&1 | tail -12
timeout 300 python tools/host_probe.py 2>&1 | grep chunk_kb | head -3
PDQ_HOST_NT=0 timeout 300 python tools/host_probe.py 2>&1 | grep chunk_kb | head -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
