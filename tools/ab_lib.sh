#!/bin/bash
# A/B two builds of libppx: tools/ab_lib.sh libA.so libB.so  (bench value + R=1 launch lists)
mkdir -p gpurun_out
for rep in 1 2; do
for L in "$@"; do
  echo -n "$L rep$rep: "
  PPX_LIB=$PWD/paper_2508_00960_b200/$L timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
done
for L in "$@"; do
  PPX_LIB=$PWD/paper_2508_00960_b200/$L timeout 200 python tools/gemm_bench.py 2>&1 | head -4 | sed "s/^/$L /"
  PPX_NOGROUP=1 PPX_LIB=$PWD/paper_2508_00960_b200/$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 370 -c 400 --csv --log-file gpurun_out/launches_$L.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-tp > /dev/null 2>&1
done
