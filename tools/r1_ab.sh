#!/bin/bash
# R=1 launch shapes (C3 per-GPU kernels of an 8-GPU run, one logical rank at a time on one GPU):
# serialised ncu launch durations of one engine step per env variant.  tools/r1_ab.sh "-" "ENV=1" ...
mkdir -p gpurun_out
i=0
for V in "$@"; do
  E="$V"; [ "$E" = "-" ] && E=""
  env PPX_NOGROUP=1 $E timeout 300 python tools/engine_one.py 2 > /dev/null 2>&1 || { echo "[$V] engine_one failed"; continue; }
  cp gpurun_out/trace.json gpurun_out/trace_$i.json
  env PPX_NOGROUP=1 $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|optimizer_kernel|peer_" --csv \
    --log-file gpurun_out/r1ab_$i.csv python tools/engine_one.py 2 > /dev/null 2>&1
  python tools/step_profile.py gpurun_out/r1ab_$i.csv gpurun_out/trace_$i.json "[$V]"
  i=$((i+1))
done
