#!/bin/bash
# Round-end run on the GPU box: smoke, the whole -m gpu suite, the bench line, the reference arm, and
# the item/user-wise CCD launch list.  Outputs under gpurun_out/fin2/.
O=gpurun_out/fin2; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ccdw_launches.csv \
    python scripts/ccdw_run.py 1 40 > /dev/null 2>&1
python scripts/launch_summary.py $O/ccdw_launches.csv > $O/ccdw_launch_summary.txt 2>&1
