"""Un-graphed engine steps on one GPU (for ncu / compute-sanitizer):
python tools/engine_one.py [steps] [--config c3|small] [--group 1] [--k3 0|1] [--dtype fp32].  --group 1 launches one logical rank at a time (the per-GPU launch shapes of a run
with one logical rank per GPU, i.e. C3 on 8 GPUs).  Writes the ABI call labels of the last step
to gpurun_out/trace.json."""
import argparse, json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_00960_b200.engine import PhantomEngine
import bench

ap = argparse.ArgumentParser()
ap.add_argument("steps", type=int, nargs="?", default=1)
ap.add_argument("--config", default="c3")
ap.add_argument("--group", type=int, default=0)
ap.add_argument("--k3", default="auto")
ap.add_argument("--dtype", default="bf16")
args = ap.parse_args()
cfg = dict(n=512, p=4, k=64, layers=3, batch=256) if args.config == "small" else bench.CONFIGS[args.config]
eng = PhantomEngine(cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"], lr=3e-6, group=args.group or None,
                    k3_fused=None if args.k3 == "auto" else args.k3 == "1",
                    dtype=torch.float32 if args.dtype == "fp32" else torch.bfloat16)
xs, ts = bench.make_data(eng, 1, cfg) if args.dtype == "bf16" else (
    [torch.randn((eng.B, eng.s), device="cuda") for _ in range(eng.R)],
    [torch.randn((eng.B, eng.s), device="cuda").clamp_min(0) for _ in range(eng.R)])
for par in (0, 1):
    eng.set_batch(xs, ts, par)
for _ in range(args.steps):
    eng.step(graph=False)
print("loss", eng.read_loss())
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"steps": args.steps, "trace": eng.trace}, open(os.path.join(ROOT, "gpurun_out", "trace.json"), "w"))
eng.close()
