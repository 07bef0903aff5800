for v in 0 1 2 3 4; do echo "== yahoo flat variant $v"; PMF_FLAT_VARIANT=$v CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
