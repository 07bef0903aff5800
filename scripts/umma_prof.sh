# timing-experiment run of the PMF_UMMA_PROFILE variant (per-warp wait cycles of CTA 0)
mkdir -p gpurun_out
cp paper_1511_02433_b200/libpmf_gpu.so /tmp/keep.so
cp scripts/_variants/libpmf_gpu_${1:-prof}.so paper_1511_02433_b200/libpmf_gpu.so
timeout 120 python bench.py --config ${2:-netflix-als} --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/uprof.json 2> gpurun_out/uprof.err
cp /tmp/keep.so paper_1511_02433_b200/libpmf_gpu.so
grep umma-prof gpurun_out/uprof.err | tail -32 > gpurun_out/uprof.txt
