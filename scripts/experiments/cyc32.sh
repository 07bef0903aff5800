timeout 900 python -m pytest tests -q -m gpu -x -k "als or adapter" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('als', d['als'])"
