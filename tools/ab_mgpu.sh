#!/bin/bash
N=$1
run() { echo -n "$1: "; env $2 timeout -k 10 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $3 bench.py --gpus $N --no-cpu-baseline --no-tp --no-e2e 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3))"; }
run halves2 "PPX_HALVES=2" 29601
run halves1 "PPX_HALVES=1" 29602
run halves2b "PPX_HALVES=2" 29603
