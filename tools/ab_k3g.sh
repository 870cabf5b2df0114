# Same-box A/B: error compression inside the first weight-gradient launch of each layer on one GPU
# (k3_grouped, default) vs its own launch (PPX_NO_K3G=1); parity tests of the new default first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_scale_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/k3g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/k3g_tests.log
for r in 1 2 3; do
  for cfg in c3 c2; do
    timeout 300 python tools/step_time.py --config $cfg --steps 30 --reps 2 2>/dev/null | tail -1
    PPX_NO_K3G=1 timeout 300 python tools/step_time.py --config $cfg --steps 30 --reps 2 2>/dev/null | tail -1
  done
done | tee gpurun_out/ab_k3g.txt
