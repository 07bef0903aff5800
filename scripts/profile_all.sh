#!/bin/bash
# Round profile set (run on the GPU box): launch lists + ncu --set full captures + CTA balance.
# Outputs under gpurun_out/prof/; summaries are copied into profiles/ by hand.
set -x
O=gpurun_out/prof; mkdir -p $O
# launch lists (per-launch device time, cold-cache serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_netflix_k40_1iter.csv python scripts/profile_run.py --iters 1 --als 1 > $O/launches_netflix.log 2>&1
python scripts/launch_summary.py $O/launches_netflix_k40_1iter.csv > $O/launch_summary_netflix.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_yahoo_k4_1iter.csv python scripts/profile_run.py --config yahoo-ccdpp --k 4 > $O/launches_yahoo.log 2>&1
python scripts/launch_summary.py $O/launches_yahoo_k4_1iter.csv > $O/launch_summary_yahoo.txt
# full captures: Netflix sweeps (promote u, promote v, plain u, plain v), Yahoo flat plain u/v, ALS
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 4 -o $O/netflix_sweeps python scripts/profile_run.py --k 2 > $O/ncu_netflix.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flat_kernel -s 6 -c 2 -o $O/yahoo_flat python scripts/profile_run.py --config yahoo-ccdpp --k 2 > $O/ncu_yahoo.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:als_gram -c 2 -o $O/als python scripts/profile_run.py --iters 0 --als 1 > $O/ncu_als.log 2>&1
for r in netflix_sweeps yahoo_flat als; do python scripts/ncu_summary.py $O/$r.ncu-rep > $O/ncu_$r.txt 2>&1; done
# per-CTA balance
timeout 600 python scripts/profile_run.py --cta --config netflix-ccdpp > $O/cta_netflix.txt 2>&1
timeout 600 python scripts/profile_run.py --cta --config yahoo-ccdpp > $O/cta_yahoo.txt 2>&1
ls -la $O
