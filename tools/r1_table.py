"""Per-kernel table of the 2nd step of `PPX_NOGROUP=1 tools/engine_one.py 2` (R=1 launch shapes of
an 8-GPU C3 run, emulated on one GPU) from an ncu gpu__time_duration launch list.
python tools/r1_table.py launches.csv [label]"""
import collections, csv, io, sys

txt = open(sys.argv[1]).read()
rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
ours = [r for r in rows if r["Kernel Name"].split("(")[0].split("<")[0].strip() in
        ("gemm_pair_kernel", "gemm_kernel", "optimizer_kernel", "peer_signal_kernel", "peer_wait_kernel")]
n = len(ours) // 2
step = ours[n:]
L, R = 8, 8
lab = ["compress"] * R
for l in range(L - 1):
    lab += ["fwd"] * R + ["compress"] * R
lab += ["fwd_loss"] * R
for l in range(L - 1, -1, -1):
    lab += ["errc"] * R
    lab += ["wgrad"] * (R if l == L - 1 else 2 * R) if False else ["wgrad"] * (len([0]) and 0)
    lab = lab  # wgrad count is data dependent; classify by position below
# position-independent classification: use grid + order is fragile; print raw sequence summary instead
agg = collections.OrderedDict()
tot = 0
for r in step:
    key = (r["Kernel Name"].split("(")[0][-20:], r["Grid Size"])
    t = float(r["Metric Value"]) / 1e3
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += t
    tot += t
print(f"== {sys.argv[2] if len(sys.argv) > 2 else ''}: {len(step)} launches, {tot:.1f} us per step (8 ranks serial)")
