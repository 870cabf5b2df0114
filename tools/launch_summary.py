"""Summarise an ncu `gpu__time_duration.sum` launch list (csv) of `bench.py --steps 1 --warmup 3`:
picks the last complete training step (the timed graph replay) of our kernels and prints the per-kernel
share table.  python tools/launch_summary.py launches.csv [launches_per_step]"""
import csv, io, sys

txt = open(sys.argv[1]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
ours = [r for r in rows if "ppx" in r["Kernel Name"] or "gemm" in r["Kernel Name"]]
print("all launches", len(rows), "ours", len(ours))
per = int(sys.argv[2]) if len(sys.argv) > 2 else None
for i, r in enumerate(ours[:per or 0]):
    print(i, r["Kernel Name"][:60], r["Grid Size"], r["Metric Value"])
