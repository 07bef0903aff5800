mkdir -p gpurun_out
for cfg in netflix-ccdpp yahoo-ccdpp; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$cfg.csv python scripts/profile_run.py --config $cfg --k 4 > gpurun_out/l_$cfg.log 2>&1
  python scripts/launch_summary.py gpurun_out/l_$cfg.csv > gpurun_out/ls_$cfg.txt 2>&1; cat gpurun_out/ls_$cfg.txt
done
PMF_PANEL_ARRAYS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_old.csv python scripts/profile_run.py --config netflix-ccdpp --k 4 > gpurun_out/l_old.log 2>&1
python scripts/launch_summary.py gpurun_out/l_old.csv
timeout 600 python scripts/profile_run.py --cta --config yahoo-ccdpp > gpurun_out/cta_yahoo.txt 2>&1; cat gpurun_out/cta_yahoo.txt
