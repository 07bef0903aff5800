for m in 8 32 64; do echo "== yahoo steal_min $m"; PMF_STEAL_MIN=$m CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
