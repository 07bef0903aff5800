mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t9.log; tail -3 gpurun_out/t9.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-als 2> gpurun_out/b9.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('netflix', d['value'], d['roofline']['usweep'], d['roofline']['vsweep'])"; grep layout gpurun_out/b9.err
timeout 900 python bench.py --config yahoo-ccdpp --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2> gpurun_out/y9.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('yahoo', d['value'], d['roofline']['usweep'], d['roofline']['vsweep'], d['quality'])"; grep layout gpurun_out/y9.err
