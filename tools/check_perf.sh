#!/bin/bash
# GPU tests + R=1 launch list + 1-GPU bench (for a kernel change)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
PPX_NOGROUP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_pair -c 176 --csv \
    --log-file gpurun_out/epi_${1:-new}.csv python tools/engine_one.py 1 > /dev/null 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
