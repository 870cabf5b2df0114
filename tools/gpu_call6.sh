mkdir -p gpurun_out
for g in 1 0; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 tools/mp_tp_parity.py --dtype fp32 --graph $g 2>&1 | grep worst | cut -c1-300; done > gpurun_out/tp3.log
for spec in "recurrence --group 1" "error --group 1" "error --group 1 --noaccum" "forward --group 1" "bwd --group 1 --k3 0" "wgrad_errors --group 1" "wgrad" "recurrence" "forward"; do
  echo "== $spec" >> gpurun_out/stats6.txt
  PPX_LIB=$PWD/paper_2508_00960_b200/libppx_stats.so PPX_DEBUG_STATS=1 timeout 200 python tools/kernel_probe.py $spec --iters 2 2>&1 | grep "ppx stats\|kind" | tail -3 >> gpurun_out/stats6.txt
done
for spec in "error --group 1" "error --group 1 --noaccum"; do PPX_NO_SPAN=1 timeout 200 python tools/kernel_probe.py $spec; done > gpurun_out/probe6_nospan.jsonl 2>&1
timeout 200 python tools/kernel_probe.py error --group 1 --noaccum > gpurun_out/probe6_noaccum.jsonl 2>&1
echo done
