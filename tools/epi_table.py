"""Per-launch-kind mean times (us) of R=1 launch lists: python tools/epi_table.py a.csv b.csv ..."""
import csv, sys
def load(p):
    lines = [l for l in open(p) if l.startswith('"')]
    return [float(r["Metric Value"].replace(",", "")) / 1000 for r in csv.DictReader(lines) if r["Metric Name"] == "gpu__time_duration.sum"]
V = {p.split("/")[-1]: load(p) for p in sys.argv[1:]}
names = {"compress": range(0, 8), "fwd": range(8, 16), "loss": range(120, 128), "B1": range(128, 136),
         "wgrad7": range(136, 144), "dgrad7": range(144, 152), "B1_6": range(152, 160), "wgrad6": range(160, 168),
         "dgrad6": range(168, 176)}
print(f"{'':10s}" + "".join(f"{v[:14]:>15s}" for v in V))
for n, r in names.items():
    print(f"{n:10s}" + "".join(f"{sum(V[v][i] for i in r) / len(r):15.1f}" for v in V))
