#!/bin/bash
# same-box A/B: coalesced (smem-staged) bf16 epilogue stores vs the per-lane row stores
for rep in 1 2; do
  for v in "" scatter; do
    for spec in "recurrence" "recurrence --group 1" "forward" "forward --group 1" "error" "wgrad_errors --group 1"; do
      echo -n "[$v] $spec: "
      PPX_DEBUG_EPI=$v timeout 200 python tools/kernel_probe.py $spec 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
    done
  done
done
