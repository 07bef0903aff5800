mkdir -p gpurun_out
for pa in 1 3; do
PMF_PANEL_ARRAYS=$pa timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 4 -c 4 -o gpurun_out/nf_pa$pa python scripts/profile_run.py --k 2 > gpurun_out/nf_pa$pa.log 2>&1; tail -2 gpurun_out/nf_pa$pa.log
done
