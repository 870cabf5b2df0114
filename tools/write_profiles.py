"""Summarise this round's GPU evidence (gpurun_out/ev_*, mg_*) into profiles/ (tracked):

  profiles/r2_bench_*.json       the bench lines (1 GPU, 2 / 4 GPUs, C2 / C4 / C5)
  profiles/r2_launches_*.txt     ncu launch-list share tables of one eager C3 step (grouped N=1 and
                                 one logical rank per launch), paired with the engine's ABI trace
  profiles/r2_ncu_*.csv          selected ncu --set full metrics of each launch kind (step shapes)
  profiles/traffic.json          DRAM bytes per launch of each kind, stamped with the commit
  profiles/r2_summary.md         the tables quoted in DESIGN.md

    python tools/write_profiles.py [commit]
"""
import csv, glob, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
COMMIT = sys.argv[1] if len(sys.argv) > 1 else subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT,
                                                              capture_output=True, text=True).stdout.strip()
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpc__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__cluster_dim_x", "sm__cycles_active.avg"]
CALL_OF = {"forward": "ppx_forward_fused", "wgrad": "ppx_wgrad", "recurrence": "ppx_backward_delta_n",
           "error": "ppx_error_phantoms_n", "wgrad_errors": "ppx_backward_wgrad_errors",
           "forward___group_1": "ppx_forward_n",
           "wgrad_errors___group_1": "ppx_backward_wgrad_errors (R=1)",
           "recurrence___group_1": "ppx_backward_delta_n (R=1)",
           "bwd___group_1___k3_0": "ppx_backward_fused"}   # tags: the probe spec with ' -' -> '_' (evidence.sh)


def raw_metrics(path):
    rows = list(csv.reader(io.StringIO(open(path).read())))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if h in KEYS}


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    os.makedirs(P, exist_ok=True)
    md = [f"# Round 2 — B200 evidence (commit {COMMIT})", ""]
    for src in sorted(glob.glob(os.path.join(G, "ev_bench.json")) + glob.glob(os.path.join(G, "mg_c*.json")) +
                      glob.glob(os.path.join(G, "ev2_*.json"))):
        try:
            line = json.loads(open(src).read().strip().splitlines()[-1])
        except Exception:
            continue
        name = os.path.basename(src).replace("ev_bench", "c3_n1").replace("mg_", "").replace("ev2_", "")
        json.dump(line, open(os.path.join(P, f"r2_bench_{name}"), "w"), indent=1)
        md.append(f"* `r2_bench_{name}`: value {line.get('value')} {line.get('unit')}, "
                  f"ms/step {line.get('ms_per_step')}, clocks {line.get('clocks', {}).get('sm_mhz')} MHz")
    md.append("")
    for g in ("8", "1"):
        lst, tr = os.path.join(G, f"ev_launches_g{g}.csv"), os.path.join(G, f"ev_trace_g{g}.json")
        if os.path.exists(lst) and os.path.exists(tr):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_step_table.py"), lst, tr,
                                  f"C3 eager step, group={g}"], capture_output=True, text=True).stdout
            open(os.path.join(P, f"r2_launches_g{g}.txt"), "w").write(out)
            md += ["```", out.rstrip(), "```", ""]
    traffic = {}
    md += ["| launch (step shapes) | ncu us | SM MHz | tensor pipe % active | DRAM MB / launch |", "|---|---|---|---|---|"]
    for path in sorted(glob.glob(os.path.join(G, "ev_full_*.raw.csv"))):
        tag = os.path.basename(path)[len("ev_full_"):-len(".raw.csv")]
        m = raw_metrics(path)
        if not m:
            continue
        with open(os.path.join(P, f"r2_ncu_{tag}.csv"), "w") as f:
            w = csv.writer(f)
            w.writerow(["metric", "value", "unit"])
            for k in KEYS:
                if k in m:
                    w.writerow([k, m[k][0], m[k][1]])
        dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
        call = CALL_OF.get(tag, tag)
        shape = "R=1 (one logical rank per launch)" if "group_1" in tag else "R=8 (grouped, N=1)"
        traffic.setdefault(call, {"dram_bytes_per_launch": dram, "commit": COMMIT, "shape": f"C3, {shape}"})
        md.append(f"| {call} ({shape}) | {m['gpu__time_duration.sum'][0]} | "
                  f"{float(m['gpc__cycles_elapsed.avg.per_second'][0]) * (1000 if m['gpc__cycles_elapsed.avg.per_second'][1] == 'Ghz' else 1):.0f} | "
                  f"{m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'][0]} | {dram / 1e6:.1f} |")
    json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
    for f in sorted(glob.glob(os.path.join(G, "cmp_*.json"))):
        json.dump(json.load(open(f)), open(os.path.join(P, "r2_" + os.path.basename(f)), "w"), indent=1)
    cli_dir = os.path.join(G, "cmp_cli_acceptance")
    if os.path.isdir(cli_dir):
        os.makedirs(os.path.join(P, "r2_cli_compare_acceptance"), exist_ok=True)
        for f in os.listdir(cli_dir):
            open(os.path.join(P, "r2_cli_compare_acceptance", f), "w").write(open(os.path.join(cli_dir, f)).read())
    for f in ("epi_ab.txt", "tp_probe.txt", "sanitize_summary.txt", "mgpu_ab.jsonl"):
        if os.path.exists(os.path.join(G, f)):
            md += ["", f"## {f}", "```", open(os.path.join(G, f)).read().rstrip(), "```"]
    open(os.path.join(P, "r2_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
