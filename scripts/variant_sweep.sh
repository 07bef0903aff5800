#!/bin/bash
# Times one CCD++ outer iteration (CUDA graph) and the per-sweep split for each launch variant.
for v in ${@:-0 1 2 3}; do
  echo "== PMF_SWEEP_VARIANT=$v"
  if [ "$v" = default ]; then unset PMF_SWEEP_VARIANT; else export PMF_SWEEP_VARIANT=$v; fi
  python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_1511_02433_b200 as P
train, probe, A = bench.make_data("netflix-ccdpp")
ctx = P.Context(A)
ctx.ccdpp_begin(P.CcdConfig(k=40, lam=0.05, outer_iters=1, inner_iters=15, seed=1))
ctx.ccdpp_iterate(2)
print("graph iter s:", [round(x, 4) for x in ctx.ccdpp_iterate(2)])
ctx.set_profiling(True); ctx.ccdpp_iterate(1); st = ctx.kernel_stats()
print("u %.1f us  v %.1f us (avg per launch incl. finalize)" % (1e3 * st["usweep_ms"] / st["usweep_launches"], 1e3 * st["vsweep_ms"] / st["vsweep_launches"]))
for side in (0, 1):
    clk, _ = ctx.debug_sweep_profile(side, False)
    d = (clk[:, 1] - clk[:, 0]) / 1e3
    print(f"side {side} plain: kernel {(clk[:,1].max()-clk[:,0].min())/1e3:.1f} us  CTA min {d.min():.1f} avg {d.mean():.1f} max {d.max():.1f}")
PY
done
