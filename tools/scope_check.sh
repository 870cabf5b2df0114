# FP32 operand-cache tests + engine / GEMM tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tf32_scope_gpu.py tests/test_engine_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/scope_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/scope_tests.log
