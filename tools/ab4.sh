#!/bin/bash
run() { echo -n "$1: "; env $2 timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; }
run single ""
run pair "PPX_PAIR=1"
run single2 ""
run pair2 "PPX_PAIR=1"
