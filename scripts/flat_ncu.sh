# ncu --set full of flat sweeps (Yahoo-Music shape, one iteration at k = 4); $1 = kernel regex
mkdir -p gpurun_out
timeout 600 ncu --kernel-name-base demangled --set full --import-source on --clock-control none -k "regex:${1:-flat_kernel}" -s ${2:-0} -c ${3:-2} -o gpurun_out/prof_flat -f python scripts/profile_run.py --config yahoo-ccdpp --iters 1 --k 4 > gpurun_out/flat_ncu.log 2>&1
