timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-als 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ingest'])"
