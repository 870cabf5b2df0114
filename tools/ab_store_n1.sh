#!/bin/bash
# same-box A/B at N=1 of the coalesced bf16 epilogue stores vs per-lane row stores (PPX_DEBUG_EPI=scatter)
for rep in 1 2 3; do
  for v in "" scatter; do
    PPX_DEBUG_EPI=$v timeout 300 python tools/step_time.py --config c3 --steps 40 --reps 2 2>/dev/null | grep config
  done
done
