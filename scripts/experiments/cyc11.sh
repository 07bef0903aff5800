mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 2 -o gpurun_out/yahoo_sweeps python scripts/profile_run.py --config yahoo-ccdpp --k 2 > gpurun_out/yahoo_ncu.log 2>&1; tail -2 gpurun_out/yahoo_ncu.log
