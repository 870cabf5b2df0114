"""FP32 tier (3xTF32): GEMM-kernel time of each operand majorness at a weight-gradient shape
(M = N = 2048, K = 8192), for the ncu launch list (splits and GEMMs are separate launches):

    ncu --metrics gpu__time_duration.sum --csv --log-file l.csv python tools/tf32_layout_probe.py
    python tools/tf32_layout_probe.py --table l.csv
"""
import csv, io, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
COMBOS = [(False, False), (False, True), (True, False), (True, True)]
REPS = 3

if len(sys.argv) > 2 and sys.argv[1] == "--table":
    txt = open(sys.argv[2]).read()
    rows = [r for r in csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])) if r.get("Metric Name") == "gpu__time_duration.sum"]
    g = [float(r["Metric Value"].replace(",", "")) for r in rows if "gemm" in r["Kernel Name"]]
    sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(rows[0]["Metric Unit"], 1.0)
    M = N = 2048; K = 8192
    for i, (ta, tb) in enumerate(COMBOS):
        t = min(g[i * REPS:(i + 1) * REPS]) * sc
        print(f"A {'MN' if ta else 'K '}-major, B {'K ' if tb else 'MN'}-major: {t:8.1f} us  "
              f"{3 * 2 * M * N * K / t / 1e6:7.1f} TF/s (tf32, 3 passes)")
    sys.exit(0)

import torch
from paper_2508_00960_b200 import kernels
M = N = 2048; K = 8192
for ta, tb in COMBOS:
    a = torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    for _ in range(REPS):
        kernels.gemm(a, b, ta, tb, out=out)
torch.cuda.synchronize()
print("ok")
