# FP32-tier (3xTF32) evidence: GEMM tests, operand-majorness probe, fp32 engine parity tests,
# split-pass share of an eager C1 / C2 step and the C2 fp32 bench line.  Outputs: gpurun_out/f32_*
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/f32_gemm_tests.log 2>&1; echo "gemm tests rc=$?"; tail -2 gpurun_out/f32_gemm_tests.log
timeout 120 python tools/tf32_layout_probe.py > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f32_layout.csv \
  python tools/tf32_layout_probe.py > /dev/null 2>&1; python tools/tf32_layout_probe.py --table gpurun_out/f32_layout.csv | tee gpurun_out/f32_layout.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "fp32 or f32 or golden or tf32 or infer" > gpurun_out/f32_tests.log 2>&1; echo "fp32 tests rc=$?"; tail -2 gpurun_out/f32_tests.log
bash tools/fp32_split.sh
timeout 300 python bench.py --config c2 --dtype fp32 --steps 10 --warmup 3 > gpurun_out/f32_bench_c2.json 2> gpurun_out/f32_bench_c2.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/f32_bench_c2.json'));print(d['value'],d['ms_per_step'],d['roofline'].get('frac_of_tier_ceiling'))"
