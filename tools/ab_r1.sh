#!/bin/bash
# same-box A/B of the R=1 fused error + weight-gradient launch: priority classes, slot pairs
for rep in 1 2; do
  for env in "" "PPX_AB_NO_PRIO=1" "PPX_AB_NO_ERROR_PAIRS=1" "PPX_AB_NO_PRIO=1 PPX_AB_NO_ERROR_PAIRS=1"; do
    echo -n "[$env] "
    env $env timeout 200 python tools/kernel_probe.py wgrad_errors --group 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
  done
  echo -n "[bwd_fused plan, wgrad+recurrence] "
  timeout 200 python tools/kernel_probe.py bwd --group 1 --k3 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
  echo -n "[bwd_fused plan, error alone] "
  timeout 200 python tools/kernel_probe.py error --group 1 --k3 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
done
