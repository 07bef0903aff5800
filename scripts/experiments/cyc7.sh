for pa in 3 1; do echo "== netflix PANEL_ARRAYS=$pa"; PMF_PANEL_ARRAYS=$pa CONFIG=netflix-ccdpp K=40 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
for pa in 1; do echo "== yahoo PANEL_ARRAYS=$pa"; PMF_PANEL_ARRAYS=$pa CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
