"""Pair an ncu gpu__time_duration launch list of `tools/engine_one.py S` with the engine's ABI call
trace (gpurun_out/trace.json) and print per-call-kind totals for the LAST step.
python tools/step_profile.py launches.csv [trace.json] [label]"""
import collections, csv, io, json, sys

txt = open(sys.argv[1]).read()
tr = json.load(open(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.json"))
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
KN = ("gemm_pair_kernel", "gemm_kernel", "optimizer_kernel", "peer_signal_kernel", "peer_wait_kernel")
ours = [r for r in rows if any(r["Kernel Name"].startswith(k) or ("::" + k) in r["Kernel Name"] for k in KN)]
trace = tr["trace"]
step = ours[len(ours) - len(trace):]
agg = collections.OrderedDict()
tot = 0.0
for name, r in zip(trace, step):
    t = float(r["Metric Value"]) / 1e3
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
    tot += t
label = sys.argv[3] if len(sys.argv) > 3 else ""
print(f"== {label} {len(trace)} launches/step ({len(ours)} ours total), sum {tot:.1f} us")
for name, (c, t) in agg.items():
    print(f"   {name:24s} x{c:3d}  {t:9.1f} us  {100 * t / tot:5.1f}%  ({t / c:.1f} us each)")
