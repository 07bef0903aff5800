mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:als_gram_tc -c 2 -o gpurun_out/prof_als -f python scripts/als_k_check.py ${1:-40} 1 > gpurun_out/ncu_als.log 2>&1
