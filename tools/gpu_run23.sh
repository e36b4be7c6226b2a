timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "property or instrumented or adversary" 2>&1 | tail -3
