# launch list (ncu, one Netflix iteration at k = 4) of the default library and each scripts/_variants/*.so
mkdir -p gpurun_out
cp paper_1511_02433_b200/libpmf_gpu.so /tmp/keep.so
for v in default scripts/_variants/libpmf_gpu_*.so; do
  [ "$v" != default ] && cp $v paper_1511_02433_b200/libpmf_gpu.so
  timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python scripts/profile_run.py --iters 1 --k 4 ${PRARGS} > /dev/null 2>&1
  echo "== $(basename $v)"; python scripts/launch_summary.py /tmp/l.csv | head -${TOPN:-5}
  cp /tmp/keep.so paper_1511_02433_b200/libpmf_gpu.so
done
