#!/bin/bash
# quick GPU check after a kernel/engine change: targeted tests, then 1-GPU (and 2-GPU) bench
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gemm_gpu.py tests/test_engine_gpu.py tests/test_multigpu_gpu.py} -x -q 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --no-tp --steps 30 > gpurun_out/q_n1.json 2>gpurun_out/q_n1.err
python -c "import json; d=json.load(open('gpurun_out/q_n1.json')); print('n1', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), round(d['e2e']['value']), d['clocks'])"
NG=$(nvidia-smi -L | wc -l)
if [ $NG -ge 2 ]; then
for N in 2 $( [ $NG -ge 4 ] && echo 4 ); do
timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) \
  bench.py --gpus $N --no-cpu-baseline --no-tp --steps 30 2>gpurun_out/q_n$N.err | grep "^{" > gpurun_out/q_n$N.json
python -c "import json; d=json.load(open('gpurun_out/q_n$N.json')); print('n$N', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d['clocks'])"
done
fi
