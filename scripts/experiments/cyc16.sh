mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t16.log; tail -3 gpurun_out/t16.log
for v in 0 1 4; do echo "== yahoo flat variant $v"; PMF_FLAT_VARIANT=$v CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
