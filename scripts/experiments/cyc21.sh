mkdir -p gpurun_out
for v in 5 6 7 0; do echo "== yahoo flat variant $v"; PMF_FLAT_VARIANT=$v CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="; done
PMF_FLAT_VARIANT=5 timeout 900 python -m pytest tests -q -m gpu -x -k "split_promote or global_gather" 2>&1 | tail -2
