#!/bin/bash
# R=1 launch lists with parts of the GEMM epilogue disabled (debug env bits)
export PPX_NOGROUP=1
for v in base NOEPI NOEPISTORE NOTMEMLD; do
  if [ $v = base ]; then E=""; else E="PPX_DEBUG_$v=1"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_pair -c 176 --csv \
    --log-file gpurun_out/epi_$v.csv python tools/engine_one.py 1 > /dev/null 2>&1
done
