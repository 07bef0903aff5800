# ALS timing of the default library and of experiment variants (scripts/_variants/libpmf_gpu_*.so)
mkdir -p gpurun_out
B="python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 5 --warmup 2"
cp paper_1511_02433_b200/libpmf_gpu.so /tmp/keep.so
for cfg in netflix-als ml10m-als; do
  echo "default $cfg $(timeout 120 $B --config $cfg 2>/dev/null | cut -c1-110)"
  echo "umma $cfg $(PMF_ALS_UMMA=1 timeout 120 $B --config $cfg 2>/dev/null | cut -c1-110)"
  for v in scripts/_variants/libpmf_gpu_*.so; do
    cp $v paper_1511_02433_b200/libpmf_gpu.so
    echo "$(basename $v) $cfg $(timeout 120 $B --config $cfg 2>/dev/null | cut -c1-110)"
    cp /tmp/keep.so paper_1511_02433_b200/libpmf_gpu.so
  done
done
