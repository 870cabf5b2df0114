#!/bin/bash
# multi-GPU A/B of env variants: tools/ab_mgpu.sh N "bench args" "-" "ENV=1" ...
mkdir -p gpurun_out
N=$1; shift; ARGS=$1; shift
for rep in 1 2; do
for V in "$@"; do
  E="$V"; [ "$E" = "-" ] && E=""
  echo -n "[N=$N $ARGS $V] "
  env $E timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) \
    bench.py --gpus $N --no-cpu-baseline --no-tp --steps 30 $ARGS 2>>gpurun_out/ab_mgpu.err | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
done
