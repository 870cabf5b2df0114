#!/bin/bash
# full ncu captures of the R=1 launch shapes: fwd, compress, loss layer, B1, wgrad, dgrad
mkdir -p gpurun_out
export PPX_NOGROUP=1
timeout 300 python tools/engine_one.py 1 || exit 1
for pair in "fwd 8" "compress 16" "loss 120" "b1 152" "wgrad 160" "dgrad 168"; do
  set -- $pair
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -s $2 -c 1 \
    -o gpurun_out/r1_$1 -f python tools/engine_one.py 1 > gpurun_out/ncu_r1_$1.log 2>&1
done
ls -la gpurun_out/
