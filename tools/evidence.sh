#!/bin/bash
# One-GPU evidence pass for profiles/: the default bench line, an ncu launch list of one eager C3
# step (grouped, N=1) and of the per-rank (R=1 shapes) step, and ncu --set full of the step's
# launch kinds at their exact shapes (tools/kernel_probe.py --ncu).  ncu runs only after the same
# command exited 0 without it.  Outputs: gpurun_out/ev_*
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
echo "bench rc=$?"
for g in 8 1; do
  timeout 300 python tools/engine_one.py 2 --group $g > /dev/null 2>&1 && cp gpurun_out/trace.json gpurun_out/ev_trace_g$g.json && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_g$g.csv \
    python tools/engine_one.py 2 --group $g > gpurun_out/ev_ncu_list_g$g.log 2>&1
  echo "launch list g$g rc=$?"
done
for spec in "forward" "wgrad" "wgrad_errors" "recurrence" "forward --group 1" "wgrad_errors --group 1" "recurrence --group 1" "bwd --group 1 --k3 0"; do
  tag=$(echo $spec | tr ' -' '__')
  timeout 200 python tools/kernel_probe.py $spec > gpurun_out/ev_probe_$tag.json 2>&1 && \
  timeout 400 ncu --set full --import-source on --clock-control none --profile-from-start off -f -o gpurun_out/ev_full_$tag \
    python tools/kernel_probe.py $spec --ncu > gpurun_out/ev_ncu_$tag.log 2>&1
  echo "$spec rc=$?"
  # keep the evidence small (gpurun returns <= 64 MiB): raw metrics + details as text; only the
  # dominant kernel's (wgrad, N=1) report itself is kept
  ncu -i gpurun_out/ev_full_$tag.ncu-rep --page raw --csv > gpurun_out/ev_full_$tag.raw.csv 2>/dev/null
  ncu -i gpurun_out/ev_full_$tag.ncu-rep --page details > gpurun_out/ev_full_$tag.details.txt 2>/dev/null
  [ "$tag" = "wgrad_errors" ] || rm -f gpurun_out/ev_full_$tag.ncu-rep
done
du -sh gpurun_out
