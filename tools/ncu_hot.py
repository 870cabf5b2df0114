"""Top SASS lines by warp-stall samples of an ncu report: python tools/ncu_hot.py rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
print("total samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:n]:
    print(f"{r[iS]:>6s} {r[iE]:>8s} {r[0][-5:]} {r[1][:100]}")
