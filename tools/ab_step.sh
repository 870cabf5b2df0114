#!/bin/bash
# A/B env variants on the C3 1-GPU step: interleaved bench runs + serialised ncu launch durations
# of one eager grouped step (clock-independent-ish).  tools/ab_step.sh "-" "ENV=1" ...
mkdir -p gpurun_out
run() { E="$1"; [ "$E" = "-" ] && E=""; env $E timeout 300 python bench.py --no-cpu-baseline --no-tp --no-e2e --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for V in "$@"; do echo -n "[$V] "; run "$V"; done
done
i=0
for V in "$@"; do
  E="$V"; [ "$E" = "-" ] && E=""
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ppx --csv \
    --log-file gpurun_out/abs_$i.csv python tools/engine_one.py 2 > /dev/null 2>&1
  python - "$V" gpurun_out/abs_$i.csv <<'PY'
import csv, io, sys
txt = open(sys.argv[2]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
n = len(rows) // 2
t = sum(float(r["Metric Value"]) for r in rows[n:]) / 1e3
print(f"[{sys.argv[1]}] ncu second step: {n} launches, {t:.1f} us")
PY
  i=$((i+1))
done
