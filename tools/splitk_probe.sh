# the layer-0 compressor-gradient split: tests + its launches in an ncu list of eager C3 steps
# with one logical rank per launch (split GEMM + summing update vs the unsplit launch)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_parity_scale_gpu.py -x -q > gpurun_out/splitk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/splitk_tests.log
for env in "" "PPX_NO_SPLITK=1"; do
  env $env timeout 300 python tools/engine_one.py 2 --group 1 > /dev/null 2>&1 && \
  env $env timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sk_launches.csv \
    python tools/engine_one.py 2 --group 1 > /dev/null 2>&1
  echo "== $env"
  python - <<'PY'
import csv, io
txt = open('gpurun_out/sk_launches.csv').read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
ours = [r for r in rows if "ppx" in r["Kernel Name"]]
# the layer-0 compressor gradient = the launches between the last ppx_reduce / recurrence and the bias optimizer of each step
idx = [i for i, r in enumerate(ours) if "optimizer_kernel" in r["Kernel Name"]]
for i in idx:
    tail = []
    j = i - 1
    while j >= 0 and ("splitk" in ours[j]["Kernel Name"] or len(tail) < 1 or "splitk" in ours[j + 1]["Kernel Name"] and "gemm" in ours[j]["Kernel Name"]):
        tail.append(ours[j]); j -= 1
        if len(tail) > 20: break
    print("  step tail:", [(r["Kernel Name"].split("(")[0][5:], r["Grid Size"], float(r["Metric Value"]) / 1e3) for r in reversed(tail)])
PY
done 2>&1 | tee gpurun_out/splitk_probe.txt
