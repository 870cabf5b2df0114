# Same-box A/B at N=2: layer-0 compressor-gradient batch split (default) vs one launch (PPX_NO_SPLITK=1)
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for r in 1 2 3; do
  timeout 300 $TR --master-port $((29900+r)) tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1
  PPX_NO_SPLITK=1 timeout 300 $TR --master-port $((29910+r)) tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1
done | tee gpurun_out/ab_splitk_n2.txt
