set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t1.log; tail -3 gpurun_out/t1.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-als > gpurun_out/b_new.json 2> gpurun_out/b_new.err; cat gpurun_out/b_new.json; grep layout gpurun_out/b_new.err
PMF_PANEL_ARRAYS=3 timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-als > gpurun_out/b_old.json 2> gpurun_out/b_old.err; cat gpurun_out/b_old.json
timeout 900 python bench.py --config yahoo-ccdpp --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/y_new.json 2> gpurun_out/y_new.err; cat gpurun_out/y_new.json; tail -5 gpurun_out/y_new.err
