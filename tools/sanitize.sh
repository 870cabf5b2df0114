#!/bin/bash
# NOTE: this pool closes compute-sanitizer (runs under it left GPUs needing a reset), so the
# script is kept for other machines; profiles/r2_sanitizer.txt records the refusal.
# compute-sanitizer (memcheck, racecheck, synccheck) over small engine steps that run every launch
# plan: grouped fused forward + grouped backward, per-rank launches with the fused error-compression
# + weight-gradient launch, the [wgrad + recurrence] fused plan, the fp32 (3xTF32) tier, and on 2 GPUs
# the NVLink fused forward + NVLink reduce-scatter (one sanitizer per rank).
# Logs: gpurun_out/sanitize_*.log ; summary lines grep'd into gpurun_out/sanitize_summary.txt
mkdir -p gpurun_out
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {   # name, tool, command...
  local name=$1 tool=$2; shift 2
  timeout 1200 $S --tool $tool "$@" > gpurun_out/sanitize_${name}_${tool}.log 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/sanitize_${name}_${tool}.log | tail -1)" \
    >> gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  run grouped $tool python tools/engine_one.py 2 --config small
  run r1k3 $tool python tools/engine_one.py 2 --config small --group 1
  run r1bwd $tool python tools/engine_one.py 2 --config small --group 1 --k3 0
  run fp32 $tool python tools/engine_one.py 2 --config small --dtype fp32
done
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  for tool in memcheck synccheck; do
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29650 --no-python $S --tool $tool python tools/mp_parity.py --dtype bf16 --p 4 --k 64 --B 256 \
      > gpurun_out/sanitize_mgpu_${tool}.log 2>&1
    echo "mgpu(fused+nvrs, 2 GPUs) $tool rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_mgpu_${tool}.log | tr '\n' ' ')" \
      >> gpurun_out/sanitize_summary.txt
  done
fi
cat gpurun_out/sanitize_summary.txt
