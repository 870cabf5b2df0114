#!/bin/bash
# multi-GPU A/B of the backward plan (k3_fused on/off) with bench.py; lines -> gpurun_out/mgpu_ab.jsonl
# usage: tools/mgpu_ab.sh N "cfg1 cfg2" reps
mkdir -p gpurun_out
N=$1; CFGS=$2; REPS=${3:-2}; PORT=29700
for rep in $(seq $REPS); do
  for cfg in $CFGS; do
    for k3 in 1 0; do
      PORT=$((PORT+1))
      out=$(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $PORT bench.py --gpus $N --config $cfg --steps 30 --warmup 5 --no-tp --no-e2e \
        --no-cpu-baseline --energy-seconds 3 --k3 $k3 2>gpurun_out/mgpu_ab_err_${N}_${cfg}_${k3}.log | tail -1)
      echo "$out" | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(json.dumps({'N': $N, 'cfg': '$cfg', 'k3': $k3, 'ms': d['ms_per_step'], 'samples_s': d['value'], 'plan': d['config']['plan'], 'step_frac_sus': d['roofline']['step_frac_of_sustained'], 'clocks': d['clocks']}))
except Exception as e: print(json.dumps({'N': $N, 'cfg': '$cfg', 'k3': $k3, 'error': str(e)}))" >> gpurun_out/mgpu_ab.jsonl
    done
  done
done
