#!/bin/bash
# One GPU evidence pass: gpu tests, smoke, 1-GPU bench (both arms), launch list, ncu full of K1.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 600 gpurun_out/bench_n1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 300 gpurun_out/bench_ref.json
[ "$1" == "noprof" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-tp > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 300 python tools/k1_probe.py && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 -o gpurun_out/k1_full -f \
  python tools/k1_probe.py > gpurun_out/ncu_k1.log 2>&1; tail -2 gpurun_out/ncu_k1.log
ls gpurun_out
