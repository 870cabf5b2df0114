#!/bin/bash
# full ncu capture of selected R=1 launches: tools/prof_one.sh tag idx [idx...]
mkdir -p gpurun_out
export PPX_NOGROUP=1
tag=$1; shift
timeout 300 python tools/engine_one.py 1 > /dev/null || exit 1
for i in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s $i -c 1 \
    -o gpurun_out/${tag}_$i -f python tools/engine_one.py 1 > gpurun_out/ncu_${tag}_$i.log 2>&1
done
