# CCD++ sweep check: GPU CCD tests, Netflix bench (no extras), launch list of one iteration (ncu, k=4)
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_ccd.py tests/test_gpu_group.py -q -x 2>&1 | tail -3 > gpurun_out/sweep_tests.log
timeout 150 python bench.py --no-extra --no-cpu-baseline --no-e2e > gpurun_out/sweep_bench.json 2> gpurun_out/sweep_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sweep_launches.csv python scripts/profile_run.py --iters 1 --k 4 > gpurun_out/sweep_launches.log 2>&1
python scripts/launch_summary.py gpurun_out/sweep_launches.csv > gpurun_out/sweep_launch_summary.txt 2>&1
