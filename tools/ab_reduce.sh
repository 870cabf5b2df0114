# NVLink reduce (ppx_reduce_received) with every source's load in flight + 1024-thread blocks vs the
# previous build (libppx_prev.so): multi-GPU parity tests, then same-box step times at N=4 and N=2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/reduce_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/reduce_tests.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
PREV=$PWD/paper_2508_00960_b200/libppx_prev.so
for r in 1 2 3; do
  for N in 4 2; do
    timeout 300 $TR --nproc-per-node $N --master-port $((29700+10*r+N)) tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1 | sed "s|^|[new] |"
    PPX_LIB=$PREV timeout 300 $TR --nproc-per-node $N --master-port $((29750+10*r+N)) tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1 | sed "s|^|[prev] |"
  done
done | tee gpurun_out/ab_reduce.txt
