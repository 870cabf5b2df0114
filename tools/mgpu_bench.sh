#!/bin/bash
# multi-GPU bench lines (N = 2, 4 on one box; N=8 emulated R=1 shapes via PPX_NOGROUP on N=1) + multi-GPU tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu_gpu.py -x -q 2>&1 | tail -2
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ $N -gt $NG ] && continue
  timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29500 + N)) bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_EXTRA} 2>gpurun_out/bench_n$N.err \
    | grep "^{" > gpurun_out/bench_n$N.json
  python -c "import json; d=json.load(open('gpurun_out/bench_n$N.json')); print($N, round(d['value']), round(d['ms_per_step'],3), d.get('tp',{}).get('value'), d['e2e']['value'], d['clocks'], d.get('pp_vs_tp'))"
done
