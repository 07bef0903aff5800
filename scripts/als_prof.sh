mkdir -p gpurun_out
B="python bench.py --config netflix-als --no-extra --no-cpu-baseline --no-e2e"
timeout 300 $B --steps 5 --warmup 2 > gpurun_out/als_base.json 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:als_umma -c 2 -o gpurun_out/prof_umma -f $B --steps 1 --warmup 1 > gpurun_out/ncu_umma.log 2>&1
cp paper_1511_02433_b200/libpmf_gpu.so /tmp/keep.so
cp scripts/_variants/libpmf_gpu_nosolve.so paper_1511_02433_b200/libpmf_gpu.so
timeout 300 $B --steps 5 --warmup 2 > gpurun_out/als_nosolve.json 2>/dev/null
cp /tmp/keep.so paper_1511_02433_b200/libpmf_gpu.so
