# full one-GPU test suite + smoke at HEAD
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_suite_1gpu.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/final_suite_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
