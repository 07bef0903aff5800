# ncu --set full of the plain flat sweeps (Yahoo-Music shape, one iteration at k = 4)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:flat_kernel -s 2 -c 2 -o gpurun_out/prof_flat -f python scripts/profile_run.py --config yahoo-ccdpp --iters 1 --k 4 > gpurun_out/flat_ncu.log 2>&1
