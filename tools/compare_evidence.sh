#!/bin/bash
# Fixed-loss PP-vs-TP evidence: the reference's acceptance comparison through our CLI (n=256, p=4,
# k=8, target 4663.4; modelled + measured energy), and the B200-scale comparison (n=8192, L=4,
# B=8192, bf16) on 1 GPU and, when present, 4 GPUs.  Outputs: gpurun_out/cmp_*
mkdir -p gpurun_out
timeout 900 python -m paper_2508_00960_b200 compare --n 256 --p 4 --k 8 --layers 2 --samples 256 --lr 1e-4 \
  --target-loss 4663.4 --max-epochs 1000 --loss-reduction mean --seed 0 --dtype fp32 --out gpurun_out/cmp_cli_acceptance \
  > gpurun_out/cmp_cli.log 2>&1; echo "cli compare rc=$?"
timeout 1200 python tools/compare_pp_tp.py --lr 1e-6 --k 128 --slack 1.10 --out gpurun_out/cmp_b200_n1_k128.json > gpurun_out/cmp_b200_n1_k128.log 2>&1; echo "b200 n1 k128 rc=$?"
for lr in 1e-6 3e-7; do
  timeout 1200 python tools/compare_pp_tp.py --lr $lr --out gpurun_out/cmp_b200_n1_lr$lr.json > gpurun_out/cmp_b200_n1_lr$lr.log 2>&1; echo "b200 n1 lr $lr rc=$?"
done
if [ "$(nvidia-smi -L | wc -l)" -ge 4 ]; then
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29851 \
    tools/compare_pp_tp.py --lr 1e-6 --out gpurun_out/cmp_b200_n4.json > gpurun_out/cmp_b200_n4.log 2>&1; echo "b200 n4 rc=$?"
fi
