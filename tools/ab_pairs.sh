#!/bin/bash
# same-box A/B of the slot-pair error tiles (PPX_AB_NO_ERROR_PAIRS) on the launches that use them
for rep in 1 2; do
  for v in "" 1; do
    for spec in "error" "wgrad_errors --group 1"; do
      echo -n "[$v] $spec: "
      PPX_AB_NO_ERROR_PAIRS=$v timeout 200 python tools/kernel_probe.py $spec 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
    done
  done
done
