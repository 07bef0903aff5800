#!/bin/bash
# One build -> measure cycle on the GPU box (run via gpurun).  Usage: scripts/gpu_cycle.sh TAG [what...]
#   what: tests | bench | benchfull | launches | ncu | smoke  (default: tests bench)
TAG=${1:-x}; shift
WHAT=${@:-tests bench}
mkdir -p gpurun_out
for w in $WHAT; do
  case $w in
    tests)  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 > gpurun_out/tests_$TAG.log; tail -3 gpurun_out/tests_$TAG.log ;;
    smoke)  timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log ;;
    bench)  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err ;;
    benchfull) timeout 1200 python bench.py > gpurun_out/benchfull_$TAG.json 2> gpurun_out/benchfull_$TAG.err; cat gpurun_out/benchfull_$TAG.json; tail -3 gpurun_out/benchfull_$TAG.err ;;
    launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_run.py --iters 1 > gpurun_out/launches_$TAG.log 2>&1; tail -2 gpurun_out/launches_$TAG.log ;;
    ncu)    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 4 -o gpurun_out/prof_$TAG python scripts/profile_run.py --iters 1 > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log ;;
  esac
done
