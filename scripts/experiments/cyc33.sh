timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for f in 1 0; do echo "== fused $f"; PMF_FUSED_FIN=$f CONFIG=netflix-ccdpp K=40 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
