timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
echo "== yahoo"; CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="
