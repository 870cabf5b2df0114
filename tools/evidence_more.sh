#!/bin/bash
# One-GPU evidence beyond C3: C4 (memory-scaled), the C5 inference sweep, the fp32 (3xTF32) tier
# at C2 and C1, and the reference arm.  Outputs: gpurun_out/ev2_*
mkdir -p gpurun_out
timeout 1200 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/ev2_c4_n1.json 2> gpurun_out/ev2_c4_n1.err; echo "c4 rc=$?"
timeout 600 python bench.py --config c5 --steps 20 > gpurun_out/ev2_c5_n1.json 2> gpurun_out/ev2_c5_n1.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c2 --dtype fp32 --steps 10 --warmup 3 --no-e2e --energy-seconds 5 > gpurun_out/ev2_c2_fp32.json 2> gpurun_out/ev2_c2_fp32.err; echo "c2 fp32 rc=$?"
timeout 600 python bench.py --config c1 --dtype fp32 --steps 50 --warmup 5 --no-e2e --energy-seconds 5 > gpurun_out/ev2_c1_fp32.json 2> gpurun_out/ev2_c1_fp32.err; echo "c1 fp32 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev2_ref.json 2> gpurun_out/ev2_ref.err; echo "ref rc=$?"
