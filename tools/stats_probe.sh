#!/bin/bash
# per-role wait / busy cycles of the launch kinds (stats build: PPX_LIB=libppx_stats.so, PPX_DEBUG_STATS=1)
for spec in "recurrence --group 1" "recurrence" "forward --group 1" "forward" "wgrad" "wgrad_errors --group 1" "error"; do
  echo "== $spec"
  PPX_LIB=$PWD/paper_2508_00960_b200/libppx_stats.so PPX_DEBUG_STATS=1 timeout 200 python tools/kernel_probe.py $spec --iters 1 2>&1 | grep "ppx stats" | tail -1
done
