# Same-box A/B of the 2-SM kernel's stage depth: K 128 x 3 stages (libppx.so) vs K 64 x 6 stages
# (libppx_pbk64.so, -DPPX_PBK=64): correctness of the variant, then C3 step times N=1 (grouped and
# one rank per launch) and per-launch-kind times (kernel_probe)
mkdir -p gpurun_out
L64=$PWD/paper_2508_00960_b200/libppx_pbk64.so
PPX_LIB=$L64 timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_parity_scale_gpu.py -x -q > gpurun_out/pbk_tests.log 2>&1; echo "pbk64 tests rc=$?"; tail -2 gpurun_out/pbk_tests.log
for r in 1 2; do
  for lib in "" "$L64"; do
    PPX_LIB=$lib timeout 300 python tools/step_time.py --steps 30 --reps 2 2>/dev/null | tail -1 | sed "s|^|[$(basename "${lib:-libppx.so}")] |"
    PPX_LIB=$lib timeout 300 python tools/step_time.py --group 1 --steps 30 --reps 2 2>/dev/null | tail -1 | sed "s|^|[$(basename "${lib:-libppx.so}")] |"
  done
done | tee gpurun_out/ab_pbk.txt
