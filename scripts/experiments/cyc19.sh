mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t19.log; tail -3 gpurun_out/t19.log
for st in 1 0; do echo "== yahoo steal=$st"; PMF_STEAL=$st CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
