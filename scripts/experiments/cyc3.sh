mkdir -p gpurun_out
CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh 0 1 2 3 4 5 6 > gpurun_out/vs_yahoo.txt 2>&1
grep -v "^\[bench\]" gpurun_out/vs_yahoo.txt
timeout 300 python scripts/profile_run.py --cta --config netflix-ccdpp > gpurun_out/cta_netflix.txt 2>&1; cat gpurun_out/cta_netflix.txt
