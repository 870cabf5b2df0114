#!/bin/bash
# Round-end check on one GPU: gpu tests + smoke, then an A/B of the tile-planner env knobs at C3 N=1.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; tail -2 gpurun_out/pytest_gpu2.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { E="$1"; [ "$E" = "-" ] && E=""; env $E timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for V in - PPX_QBAL=0.9 PPX_K3_PERRANK=1 PPX_NO_TAILSPLIT=1; do echo -n "[$V] "; run "$V"; done
done
