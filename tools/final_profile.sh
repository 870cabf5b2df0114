#!/bin/bash
# Round-end evidence on ONE GPU: bench (both arms), per-launch ncu list of one C3 step (grouped,
# N=1), ncu --set full of the dominant kernel (K1), and the R=1 launch list (8-GPU per-GPU shapes).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; tail -c 300 gpurun_out/final_bench_n1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.json 2>&1; tail -c 200 gpurun_out/final_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python tools/engine_one.py 2 > /dev/null 2>&1; cp gpurun_out/trace.json gpurun_out/final_trace.json
python tools/step_profile.py gpurun_out/final_launches.csv gpurun_out/final_trace.json "N=1 grouped (R=8)"
timeout 300 python tools/k1_probe.py > /dev/null && timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:gemm -s 2 -c 1 -o gpurun_out/final_k1 -f python tools/k1_probe.py > gpurun_out/final_k1.log 2>&1; tail -1 gpurun_out/final_k1.log
PPX_NOGROUP=1 timeout 300 python tools/engine_one.py 2 > /dev/null 2>&1; cp gpurun_out/trace.json gpurun_out/final_trace_r1.json
PPX_NOGROUP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_r1.csv \
  python tools/engine_one.py 2 > /dev/null 2>&1
python tools/step_profile.py gpurun_out/final_launches_r1.csv gpurun_out/final_trace_r1.json "R=1 shapes (per-GPU kernels of N=8)"
