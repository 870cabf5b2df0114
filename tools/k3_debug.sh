# the failing k3 run used lr 3e-3: does the separate-launch plan diverge there too?
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
i=0
for args in "--k3 1" "--k3 auto" "--k3 auto --fused 0 --nvrs 0"; do
  i=$((i+1))
  echo "== lr 3e-3 $args"
  PPX_AB_K3_PAIRS=1 timeout 150 $TR --master-port $((29980+i)) tools/mp_parity.py --dtype bf16 --p 8 --k 64 --B 256 --fused 1 --nvrs 1 $args 2>&1 | grep -E "TrainingError|pass|Error" | head -2 | grep -o -E 'TrainingError.*|"pass": [a-z]*|"losses": \[[^]]*\]|"oracle": \[[^]]*\]'
done 2>&1 | tee gpurun_out/k3_debug3.txt
