# N=2 (4 logical ranks per GPU): error compression + weight gradients as one launch with slot pairs
# (k3_fused=1) vs separate launches (default before): parity through mp_parity, then same-box A/B
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 29931 tools/mp_parity.py --dtype bf16 --p 8 --k 64 --B 256 --fused 1 --nvrs 1 --k3 1 > gpurun_out/k3n2_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/k3n2_parity.log | cut -c1-400
for r in 1 2 3; do
  timeout 300 $TR --master-port $((29940+r)) tools/step_time.py --k3 1 --steps 40 --reps 2 2>/dev/null | tail -1
  timeout 300 $TR --master-port $((29950+r)) tools/step_time.py --k3 0 --steps 40 --reps 2 2>/dev/null | tail -1
done | tee gpurun_out/ab_k3_n2.txt
