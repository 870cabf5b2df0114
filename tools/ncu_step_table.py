"""Pair an ncu launch list (`ncu --metrics gpu__time_duration.sum --clock-control none --csv`) of
`tools/engine_one.py S [...]` with the ABI-call trace the engine wrote (gpurun_out/trace.json: the
kernel-launching calls of the LAST step, in order) and print the per-call share table of that
step.  ncu's per-launch times are serialised and cold-cache: compare shares, not absolutes.

    python tools/ncu_step_table.py launches.csv trace.json [label]
"""
import collections, csv, io, json, sys

OURS = ("gemm_pair_kernel", "gemm_kernel", "optimizer_kernel", "hyper_advance_kernel", "reduce_received_kernel",
        "colsum_kernel", "cast_kernel", "output_delta_kernel", "bias_act_kernel", "relu_mask_kernel")
txt = open(sys.argv[1]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
ours = [r for r in rows if any(k in r["Kernel Name"] for k in OURS)]
trace = json.load(open(sys.argv[2]))["trace"]
label = sys.argv[3] if len(sys.argv) > 3 else ""
last = ours[-len(trace):]
agg = collections.OrderedDict()
unit = last[0]["Metric Unit"] if last else "us"
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
for call, r in zip(trace, last):
    a = agg.setdefault(call, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"].replace(",", "")) * scale
total = sum(v[1] for v in agg.values())
print(f"== {label} {len(trace)} kernel launches in the step, ncu sum {total:.1f} us")
for call, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"   {call:28s} x{n:3d} {t:10.1f} us {100 * t / total:6.1f}%  ({t / n:.1f} us each)")
