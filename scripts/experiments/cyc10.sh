mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t10.log; tail -3 gpurun_out/t10.log
for st in 1 0; do
echo "== netflix steal=$st"; PMF_STEAL=$st CONFIG=netflix-ccdpp K=40 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="
echo "== yahoo steal=$st"; PMF_STEAL=$st CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="
done
