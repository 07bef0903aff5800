# Netflix CCD++ iteration and per-CTA spread under the default vs a candidate PMF_UNIT_COST
mkdir -p gpurun_out
for m in "" "$1"; do
  if [ -n "$m" ]; then export PMF_UNIT_COST="$m"; else unset PMF_UNIT_COST; fi
  echo "== model '${m:-default}'"
  timeout 200 python scripts/profile_run.py --cta 2>&1 | grep "^side"
  for i in 1 2; do timeout 150 python bench.py --no-extra --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('value',d['value'],'v-sweep',d['roofline']['vsweep'],'clk',d['clocks']['sm_mhz'])"; done
done
