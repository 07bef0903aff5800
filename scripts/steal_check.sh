for s in "" 1; do
  if [ -n "$s" ]; then export PMF_STEAL=$s; else unset PMF_STEAL; fi
  echo "== PMF_STEAL=${s:-default}"
  timeout 200 python scripts/profile_run.py --cta 2>&1 | grep "^side"
  for i in 1 2; do timeout 150 python bench.py --no-extra --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "import json,sys;d=json.loads(sys.stdin.read());print('value',d['value'],'u',d['roofline']['usweep']['ms'],'v',d['roofline']['vsweep']['ms'],'clk',d['clocks']['sm_mhz'])"; done
done
