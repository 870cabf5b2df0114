mkdir -p gpurun_out
for c in c1 c2; do
  timeout 300 python tools/engine_one.py 1 --config $c --dtype fp32 > gpurun_out/f32_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f32_launches_$c.csv \
    python tools/engine_one.py 1 --config $c --dtype fp32 > gpurun_out/f32_ncu_$c.log 2>&1
  echo "$c rc=$?"
  python tools/kernel_share.py gpurun_out/f32_launches_$c.csv "fp32 $c eager step" > gpurun_out/f32_share_$c.txt 2>&1
  cat gpurun_out/f32_share_$c.txt
done
