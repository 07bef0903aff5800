mkdir -p gpurun_out
bash scripts/profile_all.sh > gpurun_out/profile_all.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; cat gpurun_out/bench_final.json
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
