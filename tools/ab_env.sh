#!/bin/bash
# A/B of env toggles in one session: tools/ab_env.sh "ENV_A" "ENV_B"  (use "-" for none)
mkdir -p gpurun_out
run() { E="$1"; [ "$E" = "-" ] && E=""; env $E timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for rep in 1 2 3; do
  for V in "$@"; do echo -n "[$V] "; run "$V"; done
done
i=0
for V in "$@"; do
  E="$V"; [ "$E" = "-" ] && E=""
  env PPX_NOGROUP=1 $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_pair -c 176 --csv \
    --log-file gpurun_out/ab_$i.csv python tools/engine_one.py 1 > /dev/null 2>&1
  i=$((i+1))
done
