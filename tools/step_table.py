"""Per-kernel share table of one C3 training step (N=1, 8 logical ranks grouped) from an ncu launch
list of `bench.py --steps 1 --warmup 3 --no-tp --no-e2e --no-cpu-baseline` (first eager step).
python tools/step_table.py launches.csv [first_index_of_step]"""
import collections, csv, io, sys

txt = open(sys.argv[1]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
ours = [r for r in rows if r["Kernel Name"].startswith("ppx::")]
i0 = int(sys.argv[2]) if len(sys.argv) > 2 else 11
L = 8
step = ours[i0:i0 + 104]
lab = []
lab.append("K2 compress (8 ranks grouped)")
for l in range(L - 1):
    lab += ["K1 fused forward + bias + ReLU (8 ranks)", "K2 compress (8 ranks grouped)"]
lab.append("K1 output layer + delta + loss + d bias")
for l in range(L - 1, -1, -1):
    lab += ["K3 error compression (per rank)"] * 8
    lab += ["K4/K5 weight grads + fused SGD"] * (1 if l == L - 1 else 2)
    if l > 0:
        lab.append("K6 [delta|r].[L;C] + ReLU' + d bias (8 ranks)")
lab += ["d compressor layer 0 + SGD", "bias SGD (elementwise)"]
assert len(lab) == len(step), (len(lab), len(step))
flops = {}
n, p, k, B = 16384, 8, 128, 8192
s = n // p
fl = {"K2": 8 * 2 * B * s * k, "K1 f": 8 * 2 * B * s * (s + (p - 1) * k), "K1 o": 8 * 2 * B * s * (s + (p - 1) * k),
      "K3": 2 * B * s * (p - 1) * k, "K6": 8 * 2 * B * s * (s + k)}
agg = collections.OrderedDict()
tot = 0.0
for name, r in zip(lab, step):
    t = float(r["Metric Value"]) / 1e3
    a = agg.setdefault(name, [0, 0.0, r["Grid Size"]])
    a[0] += 1
    a[1] += t
    tot += t
print(f"| kernel | grid | launches/step | us per launch | share | TFLOP/s |")
print("|---|---|---|---|---|---|")
for name, (c, t, g) in agg.items():
    f = next((v for key, v in fl.items() if name.startswith(key)), None)
    tf = f"{f / (t / c * 1e-6) / 1e12:.0f}" if f else "-"
    print(f"| {name} | {g.split(',')[0].strip('(')} | {c} | {t / c:.1f} | {100 * t / tot:.1f}% | {tf} |")
print(f"\nsum of launch durations (serialised, clocks uncapped): {tot / 1e3:.2f} ms per step")
