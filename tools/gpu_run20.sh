timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C2.desc C2.asc C2.organ C1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), d['config']['sort_ok'], d['config']['reference_digest_ok'])"; done
