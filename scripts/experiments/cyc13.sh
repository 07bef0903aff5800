CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh 2 7 8 0 6 1 2>&1 | grep -v "^\[bench\]"
