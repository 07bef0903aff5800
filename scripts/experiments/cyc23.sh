mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for t in 1 0; do PMF_ALS_TMA=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma', $t, 'als', d['als'])"; done
