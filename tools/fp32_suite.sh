mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f32_full_suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/f32_full_suite.log
bash tools/fp32_split.sh
timeout 300 python bench.py --config c2 --dtype fp32 --steps 10 --warmup 3 > gpurun_out/f32_bench_c2.json 2> gpurun_out/f32_bench_c2.err; echo "bench rc=$?"
timeout 300 python bench.py --config c1 --dtype fp32 --steps 20 --warmup 3 > gpurun_out/f32_bench_c1.json 2> gpurun_out/f32_bench_c1.err; echo "bench c1 rc=$?"
python -c "
import json
for c in ('c1','c2'):
    d=json.load(open(f'gpurun_out/f32_bench_{c}.json'));r=d['roofline'];print(c,d['value'],d['ms_per_step'],r.get('frac_of_tier_ceiling'));[print('  ',k,round(v['ms_per_step'],2),v['launches_per_step']) for k,v in r['kernels'].items()]"
