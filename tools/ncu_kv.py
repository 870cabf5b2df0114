"""Print selected raw metrics of ncu reports: python tools/ncu_kv.py rep... -- metric_substr..."""
import csv, io, subprocess, sys
args = sys.argv[1:]
sep = args.index("--") if "--" in args else len(args)
reps, keys = args[:sep], args[sep + 1:]
for rep in reps:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    for v in vals:
        print("==", rep)
        for h, u, x in zip(hdr, units, v):
            if any(k in h for k in keys):
                print(f"  {h:80s} {x:>16s} {u}")
