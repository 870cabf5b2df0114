# N=2 with the error compression inside the weight-gradient launch (now default at 4 ranks / GPU):
# the 2-GPU parity tests, then the bench line at N=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/k3n2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/k3n2_tests.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 $TR --master-port 29802 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/mg_c3_n2.json 2> gpurun_out/mg_c3_n2.err; echo "c3 n2 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/mg_c3_n2.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['clocks'],d['config']['plan'])"
