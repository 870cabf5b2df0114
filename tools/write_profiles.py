"""Summarise the round-end GPU evidence (gpurun_out/final_*) into profiles/ (tracked)."""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def ncu_raw(rep, keys):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if h in keys}


def step_table(launches, trace, label):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "step_profile.py"), launches, trace, label],
                          capture_output=True, text=True).stdout


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpc__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__grid_size", "launch__cluster_dim_x"]
k1 = ncu_raw(os.path.join(G, "final_k1.ncu-rep"), keys)
rd = float(k1["dram__bytes_read.sum"][0]) * (1e6 if k1["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if k1["dram__bytes_read.sum"][1] == "Gbyte" else 1)
wr = float(k1["dram__bytes_write.sum"][0]) * (1e6 if k1["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if k1["dram__bytes_write.sum"][1] == "Gbyte" else 1)
json.dump({"kernel": "gemm_pair_kernel as ppx_forward_update (C3 layer, one logical rank: M=8192, N=2048, K=2048+7*128)",
           "source": "ncu --set full --clock-control none (tools/final_profile.sh, k1_probe.py launch 3), dram__bytes_read.sum + dram__bytes_write.sum",
           "dram_bytes_per_launch": int(rd + wr), "algorithmic_bytes_per_launch": 52690944,
           "note": "algorithmic = Y 32 MiB + gathered phantoms 14 MiB + L 8 MiB + D 3.5 MiB read, Y_out 32 MiB written; "
                   "DRAM write < 32 MiB because the output stays L2-resident at kernel end"},
          open(os.path.join(P, "k1_traffic.json"), "w"), indent=1)
lines = ["# Round 1 (final) — B200 evidence", "",
         "Commands: `tools/final_profile.sh` on one GPU (ncu only after the same command exited 0 without it);",
         "multi-GPU lines from `bench.py` under torchrun on one 4-GPU box. Per-launch ncu times are serialised",
         "and cold-cache at uncapped clocks: compare shares, not absolutes.", "",
         "## K1 (fused forward GEMM, the roofline kernel) — ncu --set full", "", "| metric | value |", "|---|---|"]
for kk in keys:
    if kk in k1:
        lines.append(f"| {kk} | {k1[kk][0]} {k1[kk][1]} |")
lines += ["", "## One C3 training step on 1 GPU (8 logical ranks, grouped launches)", "", "```",
          step_table(os.path.join(G, "final_launches.csv"), os.path.join(G, "final_trace.json"), "N=1 grouped (R=8)").strip(),
          "```", "", "## The same step with one logical rank per launch (per-GPU kernels of an 8-GPU run; unfused forward)", "",
          "```", step_table(os.path.join(G, "final_launches_r1.csv"), os.path.join(G, "final_trace_r1.json"),
                             "R=1 shapes").strip(), "```", "", "## bench.py lines", ""]
for f in ["final_bench_n1.json", "final_bench_ref.json", "final_bench_n2.json", "final_bench_n4.json", "final_bench_c2_n4.json"]:
    path = os.path.join(G, f)
    if os.path.exists(path) and os.path.getsize(path):
        d = json.loads(open(path).read().strip().splitlines()[-1])
        keep = {k: d.get(k) for k in ("impl", "value", "ms_per_step", "n_gpus", "e2e", "roofline", "clocks", "cpu_baseline",
                                       "pp_vs_tp", "energy", "comm_bytes_per_step_per_gpu") if k in d}
        if d.get("tp"):
            keep["tp"] = {k: d["tp"].get(k) for k in ("value", "ms_per_step", "comm_bytes_per_step_per_gpu", "j_per_epoch")}
        lines += [f"### {f}", "", "```json", json.dumps(keep, indent=1), "```", ""]
        os.makedirs(P, exist_ok=True)
        open(os.path.join(P, "r1_" + f), "w").write(open(path).read())
open(os.path.join(P, "r1_final_summary.md"), "w").write("\n".join(lines) + "\n")
for src, dst in [("final_launches.csv", "r1_final_launches_n1.csv"), ("final_launches_r1.csv", "r1_final_launches_r1shapes.csv")]:
    open(os.path.join(P, dst), "w").write(open(os.path.join(G, src)).read())
print("\n".join(lines))
