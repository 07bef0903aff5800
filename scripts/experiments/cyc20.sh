for b in 220 200 192 160; do echo "== yahoo budget $b"; PMF_SMEM_BUDGET_KB=$b CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
