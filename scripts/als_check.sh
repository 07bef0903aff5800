mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_als.py tests/test_gpu_ccdw.py -q -x 2>&1 | tail -15 > gpurun_out/als_tests.log
for cfg in netflix-als ml10m-als; do
  timeout 120 python bench.py --config $cfg --no-extra --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > gpurun_out/als_$cfg.json 2> gpurun_out/als_$cfg.err
done
if [ -n "$NCU" ]; then
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:als_umma -c 2 -o gpurun_out/prof_umma -f python bench.py --config netflix-als --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_umma.log 2>&1
fi
for f in gpurun_out/als_*.json; do echo $f; cut -c1-120 $f; done
