# Round-end 4-GPU evidence at the final commit: C3 at N=2 and 4, C2 / C4 at N=4, the C5 sweep at
# N=2 and 4, per-call traces, the full GPU test suite (multi-GPU parity included) and smoke.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/mg_c3_n2.json 2> gpurun_out/mg_c3_n2.err; echo "c3 n2 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/mg_c3_n4.json 2> gpurun_out/mg_c3_n4.err; echo "c3 n4 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --config c2 --steps 20 --warmup 5 --no-tp > gpurun_out/mg_c2_n4.json 2> gpurun_out/mg_c2_n4.err; echo "c2 n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --config c4 --steps 10 --warmup 3 --no-e2e > gpurun_out/mg_c4_n4.json 2> gpurun_out/mg_c4_n4.err; echo "c4 n4 rc=$?"
for N in 2 4; do timeout 600 $TR --nproc-per-node $N --master-port $((29810+N)) bench.py --gpus $N --config c5 --steps 20 > gpurun_out/mg_c5_n$N.json 2> gpurun_out/mg_c5_n$N.err; echo "c5 n$N rc=$?"; done
for N in 2 4; do timeout 300 $TR --nproc-per-node $N --master-port $((29820+N)) tools/mp_trace.py --config c3 > gpurun_out/mg_trace_c3_n$N.txt 2>&1; echo "trace n$N rc=$?"; done
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/mg_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mg_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/mg_smoke.log 2>&1; echo "smoke rc=$?"
