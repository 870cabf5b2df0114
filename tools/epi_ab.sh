#!/bin/bash
# Which part of the epilogue bounds the short-K launches: recurrence / error compression timed
# with the ReLU'-mask read and / or the column sums dropped (PPX_DEBUG_EPI, wrong results, A/B only)
mkdir -p gpurun_out
for spec in "recurrence" "recurrence --group 1" "forward" "error"; do
  for v in "" mask colsum mask,colsum; do
    echo -n "$spec [$v] "
    PPX_DEBUG_EPI=$v timeout 200 python tools/kernel_probe.py $spec 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_launch'],1), 'us', round(d['frac_of_burst'],3))"
  done
done
