mkdir -p gpurun_out
CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh 2 1 0 3 2>&1 | grep -v "^\[bench\]" > gpurun_out/vs4_yahoo.txt; cat gpurun_out/vs4_yahoo.txt
echo "== yahoo len order"; PMF_UNIT_ORDER=len CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh 2 2>&1 | grep -v "^\[bench\]"
for v in 2 1 0 3; do echo "== netflix CSC variant $v"; PMF_SWEEP_VARIANT_CSR=1 CONFIG=netflix-ccdpp K=40 timeout 900 bash scripts/variant_sweep.sh $v 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
echo "== netflix old layout"; PMF_PANEL_ARRAYS=3 CONFIG=netflix-ccdpp K=40 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]"
