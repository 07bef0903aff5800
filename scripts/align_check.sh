#!/bin/bash
# Graph iteration time and plain-sweep split for several segment alignments (PMF_SEG_ALIGN).
for a in ${@:-4 8 16}; do
  echo "== PMF_SEG_ALIGN=$a"
  PMF_SEG_ALIGN=$a scripts/variant_sweep.sh default 2>&1 | grep -v "^\[bench\]\|^=="
done
