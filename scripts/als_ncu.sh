mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:als_umma -c 1 -o gpurun_out/prof_umma -f python bench.py --config ${1:-netflix-als} --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_umma.log 2>&1
