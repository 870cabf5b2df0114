mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_scale_gpu.py tests/test_tf32_scope_gpu.py -x -q > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/quick_tests.log
