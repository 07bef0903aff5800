# Yahoo-Music CCD++: flat-layout GPU tests and timing (default vs PMF_FLAT_RMW=1)
mkdir -p gpurun_out
PMF_FLAT_RMW=1 timeout 300 python -m pytest tests/test_gpu_ccd.py tests/test_gpu_group.py -q -x 2>&1 | tail -3
for e in 0 1; do
  PMF_FLAT_RMW=$e timeout 300 python bench.py --config yahoo-ccdpp --steps 2 --warmup 1 --no-extra --no-cpu-baseline --no-e2e > /tmp/y.json 2>/dev/null
  echo "PMF_FLAT_RMW=$e $(python3 -c "import json;d=json.load(open('/tmp/y.json'));print(d['value'], d['roofline']['whole_iteration'], d['quality'])")"
done
