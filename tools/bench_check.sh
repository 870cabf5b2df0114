# default bench line (N=1) + launch list of one eager C3 step with one logical rank per launch
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bc_bench.json 2> gpurun_out/bc_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bc_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['gpu_launches'],d['clocks']['sm_mhz']);print(d['fp32_tier']);print({k:v for k,v in d['r1_shapes'].items() if k!='kernels'})"
timeout 300 python tools/engine_one.py 2 --group 1 > /dev/null 2>&1 && cp gpurun_out/trace.json gpurun_out/bc_trace_g1.json && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bc_launches_g1.csv \
  python tools/engine_one.py 2 --group 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/kernel_share.py gpurun_out/bc_launches_g1.csv "C3 group=1, 2 eager steps" | head -12
