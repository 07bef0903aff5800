#!/bin/bash
# Round-end artefacts on the GPU box: bench lines (Netflix, Yahoo, reference arm), smoke, profile set.
set -x
mkdir -p gpurun_out/fin
timeout 900 python bench.py > gpurun_out/fin/bench_netflix.json 2> gpurun_out/fin/bench_netflix.err
timeout 1200 python bench.py --config yahoo-ccdpp --no-cpu-baseline > gpurun_out/fin/bench_yahoo.json 2> gpurun_out/fin/bench_yahoo.err
timeout 900 python bench.py --impl reference > gpurun_out/fin/bench_reference.json 2> gpurun_out/fin/bench_reference.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1
bash scripts/profile_all.sh > gpurun_out/fin/profile_all.log 2>&1
