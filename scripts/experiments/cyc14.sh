mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t14.log; tail -5 gpurun_out/t14.log
echo "== yahoo flat"; CONFIG=yahoo-ccdpp K=4 timeout 900 bash scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]" | grep -v "=="
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l14_y.csv python scripts/profile_run.py --config yahoo-ccdpp --k 4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/l14_y.csv
