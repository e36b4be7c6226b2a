timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/fallback_bench.py 28 2>&1 | grep -v k16
timeout 900 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],3), d['phase_ms'], d['config']['sort_ok'], d['config']['reference_digest_ok'])"
