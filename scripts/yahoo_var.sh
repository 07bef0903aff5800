# Yahoo-Music CCD++ seconds per iteration: default library vs each scripts/_variants/*.so
cp paper_1511_02433_b200/libpmf_gpu.so /tmp/keep.so
for v in default scripts/_variants/libpmf_gpu_*.so; do
  [ "$v" != default ] && cp $v paper_1511_02433_b200/libpmf_gpu.so
  timeout 300 python bench.py --config ${CFG:-yahoo-ccdpp} --steps 2 --warmup 1 --no-extra --no-cpu-baseline --no-e2e > /tmp/y.json 2>/dev/null
  echo "$(basename $v) $(python3 -c "import json;d=json.load(open('/tmp/y.json'));print(d['value'], d['roofline']['whole_iteration']['frac'], d['quality']['objective'], d['clocks']['sm_mhz'])")"
  cp /tmp/keep.so paper_1511_02433_b200/libpmf_gpu.so
done
