"""Un-graphed engine steps at config C3 on one GPU (for ncu). PPX_NOGROUP=1 gives R=1 launch
shapes (an 8-GPU run's per-GPU kernels, one logical rank at a time).  Writes the ABI call labels
of the last step to gpurun_out/trace.json (tools/step_profile.py pairs them with ncu launches)."""
import json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_00960_b200.engine import PhantomEngine
cfg = os.environ.get("PPX_CFG", "16384,8,128,8,8192")
n, p, k, L, B = (int(x) for x in cfg.split(","))
eng = PhantomEngine(n, p, k, L, B, lr=3e-6)
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn((B, eng.s), device="cuda", generator=g).bfloat16() for _ in range(eng.R)]
ts = [torch.randn((B, eng.s), device="cuda", generator=g).bfloat16() for _ in range(eng.R)]
for par in (0, 1):
    eng.set_batch(xs, ts, par)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for _ in range(steps):
    eng.step(graph=False)
print("loss", eng.read_loss())
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"steps": steps, "trace": eng.trace}, open(os.path.join(ROOT, "gpurun_out", "trace.json"), "w"))
eng.close()
