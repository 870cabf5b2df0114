#!/bin/bash
# same-box A/B on N GPUs: coalesced epilogue stores vs per-lane row stores (graph-replayed steps)
N=$1; PORT=29900
for rep in 1 2; do
  for v in "" scatter; do
    for cfg in c3 c2; do
      PORT=$((PORT+1))
      PPX_DEBUG_EPI=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $PORT tools/step_time.py --config $cfg 2>/dev/null | grep config
    done
  done
done
