# Same-box A/B of the layer-0 compressor-gradient split (ppx_wgrad_splitk) vs one launch
# (PPX_NO_SPLITK=1): C3 grouped (N=1) and on 2 / 4 GPUs when present
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_scale_gpu.py tests/test_tf32_scope_gpu.py -x -q > gpurun_out/splitk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/splitk_tests.log
NG=$(nvidia-smi -L | wc -l)
for r in 1 2; do
  timeout 300 python tools/step_time.py --steps 30 --reps 2 2>/dev/null | tail -1
  PPX_NO_SPLITK=1 timeout 300 python tools/step_time.py --steps 30 --reps 2 2>/dev/null | tail -1
  if [ "$NG" -ge 4 ]; then
    timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1
    PPX_NO_SPLITK=1 timeout 300 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/step_time.py --steps 40 --reps 2 2>/dev/null | tail -1
  fi
done | tee gpurun_out/ab_splitk.txt
