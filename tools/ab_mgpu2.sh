#!/bin/bash
N=$1
run() { echo -n "$1: "; env $2 timeout -k 10 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $3 bench.py --gpus $N --no-cpu-baseline --no-tp --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['step_tflops_per_gpu']))"; }
run base "PPX_COMM_SMS=0" 29601
run comm8 "PPX_COMM_SMS=8" 29602
run comm16 "PPX_COMM_SMS=16" 29603
run halves "PPX_HALVES=2" 29604
run base2 "PPX_COMM_SMS=0" 29605
