#!/bin/bash
# Item/user-wise CCD on the Netflix shape: epoch timing, the GPU tests, and a launch list of one epoch
# (gpurun_out/ccdw_launch.csv).  Usage (on the GPU box): bash scripts/ccdw_launch.sh
timeout 300 python scripts/ccdw_run.py 3 40 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_ccdw.py -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ccdw_launch.csv \
    python scripts/ccdw_run.py 1 40 > /dev/null 2>&1
python - <<'PY'
import collections, csv
rows = list(csv.reader(open("gpurun_out/ccdw_launch.csv")))
h, agg = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"][:60]].append(float(d["Metric Value"]) / 1e6)
for k, v in agg.items():
    print(f"{k:60s} n={len(v)} ms={[round(x, 3) for x in v[-4:]]}")
PY
