"""Per-CUDA-source-line warp-stall samples of an ncu report (cuda,sass view): top lines + reasons.
python tools/ncu_lines.py rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; hdr = None; agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or r[0] == "": continue   # sass rows have empty line no
    # source text may carry unescaped quotes: align the metric columns from the right
    r = r[:2] + r[len(r) - (len(hdr) - 2):]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    if r[iS] in ("-", ""): continue
    key = (fname, int(r[0]))
    st = {h[6:]: float(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("-", "")}
    agg[key] = (int(r[iS]), r[1].strip()[:70], st, int(r[hdr.index("Instructions Executed")] or 0))
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(v[2].items(), key=lambda x: -x[1])[:3]
    print(f"{v[0]:6d} {k[0][:14]:14s}:{k[1]:<4d} {v[1]:70s} inst={v[3]:<8d} {[(a, int(b)) for a, b in top]}")
