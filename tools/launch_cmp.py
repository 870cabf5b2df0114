"""Compare ncu launch lists (gpu__time_duration.sum CSVs) position by position."""
import csv, sys
def load(p):
    rows = []
    with open(p) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"][:40], r["Grid Size"], float(r["Metric Value"].replace(",", "")) / (1000.0 if r["Metric Unit"] == "nsecond" else 1.0)))
    return rows
A = [load(p) for p in sys.argv[1:]]
n = min(len(a) for a in A)
tot = [0.0] * len(A)
for i in range(n):
    vals = [a[i][2] for a in A]
    for j, v in enumerate(vals): tot[j] += v
    if i < int(sys.argv[0] and 10**9):
        print(f"{i:4d} {A[0][i][0]:40s} {A[0][i][1]:>14s} " + " ".join(f"{v:9.1f}" for v in vals))
print("total us:", " ".join(f"{t:.0f}" for t in tot))
