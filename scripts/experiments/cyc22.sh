mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_netflix.json 2> gpurun_out/bench_netflix.err; cat gpurun_out/bench_netflix.json
timeout 1500 python bench.py --config yahoo-ccdpp --no-cpu-baseline > gpurun_out/bench_yahoo.json 2> gpurun_out/bench_yahoo.err; cat gpurun_out/bench_yahoo.json; tail -3 gpurun_out/bench_yahoo.err
