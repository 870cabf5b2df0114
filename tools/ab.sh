#!/bin/bash
# A/B the GEMM code paths on the real training step (bench.py, 1 GPU, C3)
run() { echo -n "$1: "; env $2 timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; }
run default ""
run no5d "PPX_NO_5D=1"
run nopair "PPX_NO_PAIR=1"
run nopair_no5d "PPX_NO_PAIR=1 PPX_NO_5D=1"
run default2 ""
