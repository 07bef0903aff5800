mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:flat_kernel -s 6 -c 2 -o gpurun_out/yflat python scripts/profile_run.py --config yahoo-ccdpp --k 2 > gpurun_out/yflat.log 2>&1; tail -1 gpurun_out/yflat.log
