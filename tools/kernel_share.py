"""Per-kernel-name share table of an ncu launch list (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv`), e.g. of `tools/engine_one.py 1 --dtype fp32`: how much of the
step the FP32 tier's hi/lo split passes take next to its GEMMs.

    python tools/kernel_share.py launches.csv [label]
"""
import collections, csv, io, sys

txt = open(sys.argv[1]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].split("<")[0].strip()
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
total = sum(v[1] for v in agg.values())
gemm = sum(v[1] for k, v in agg.items() if "gemm" in k)
split = sum(v[1] for k, v in agg.items() if "split_tf32" in k)
print(f"== {sys.argv[2] if len(sys.argv) > 2 else ''} {len(rows)} launches, ncu sum {total:.1f} us")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"   {k[:40]:40s} x{n:4d} {t:10.1f} us {100 * t / total:6.1f}%")
if gemm:
    print(f"   split passes / GEMM time = {split / gemm:.3f}")
