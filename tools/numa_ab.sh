#!/bin/bash
# e2e A/B at C3 on 4 GPUs: ranks bound to their GPU's NVML CPU affinity (default) vs unbound.
mkdir -p gpurun_out
nvidia-smi topo -m 2>&1 | head -12; lscpu | grep -i "numa\|^CPU(s)"
run() { env $1 timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port $2 bench.py --gpus 4 --steps 20 --warmup 5 --no-cpu-baseline --no-tp 2>>gpurun_out/numa.err | grep "^{" | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],3))"; }
for rep in 1 2; do run PPX_NO_NUMA_BIND=1 $((29700+rep)); run PPX_X=0 $((29710+rep)); done
