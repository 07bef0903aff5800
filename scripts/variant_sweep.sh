#!/bin/bash
# Per-variant timing of the plain sweeps.  Usage: CONFIG=yahoo-ccdpp K=4 scripts/variant_sweep.sh 0 1 2 ...
for v in ${@:-0 1 2 3}; do
  echo "== PMF_SWEEP_VARIANT=$v"
  if [ "$v" = default ]; then :; elif [ -n "$PMF_SWEEP_VARIANT_CSR" ]; then export PMF_SWEEP_VARIANT_CSC=$v; else export PMF_SWEEP_VARIANT=$v; fi
  python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
cfg = os.environ.get("CONFIG", "netflix-ccdpp"); k = int(os.environ.get("K", "40"))
train, probe, A = bench.make_data(cfg)
ctx = P.Context(A)
ctx.ccdpp_begin(P.CcdConfig(k=k, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
ctx.ccdpp_iterate(1)
print("graph iter s:", [round(x, 4) for x in ctx.ccdpp_iterate(2)])
ctx.set_profiling(True); ctx.ccdpp_iterate(1); st = ctx.kernel_stats()
print("u %.1f us  v %.1f us (avg per launch incl. finalize)" % (1e3 * st["usweep_ms"] / st["usweep_launches"], 1e3 * st["vsweep_ms"] / st["vsweep_launches"]))
for side in (0, 1):
    clk, _ = ctx.debug_sweep_profile(side, False)
    d = (clk[:, 1] - clk[:, 0]) / 1e3
    print(f"side {side} plain: kernel {(clk[:,1].max()-clk[:,0].min())/1e3:.1f} us  CTA min {d.min():.1f} avg {d.mean():.1f} max {d.max():.1f}")
PY
done
