#!/bin/bash
export PPX_NOGROUP=1
for v in NOCOLSUM NOMASK NOSTORE2 ALL3; do
  if [ $v = ALL3 ]; then E="PPX_DEBUG_NOCOLSUM=1 PPX_DEBUG_NOMASK=1 PPX_DEBUG_NOSTORE2=1"; else E="PPX_DEBUG_$v=1"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_pair -c 176 --csv \
    --log-file gpurun_out/epi_$v.csv python tools/engine_one.py 1 > /dev/null 2>&1
done
