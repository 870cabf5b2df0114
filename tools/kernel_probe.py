"""Time (or ncu-profile) ONE launch kind of the C3 training step at its exact step shapes:

    python tools/kernel_probe.py KIND [--group 1|8] [--iters 20] [--config c3] [--ncu]

KIND: forward (fused / grouped forward), error (error compression as its own launch), wgrad
(grouped weight gradients), bwd (fused weight-gradient + recurrence launch, group=1 --k3 0),
wgrad_errors (fused error-compression + weight-gradient launch: the one-GPU default plan, or
group=1), recurrence, compress — the middle launch of
that kind in the step (--index to pick another).  The launches are issued exactly as
PhantomEngine._step_body issues them (the engine records every kernel call of an eager step with
its ABI arguments; the probe re-issues the chosen one) back to back behind a ~0.1 s device spin
(so host launch cost never starves the GPU) and timed with CUDA events.  --ncu brackets ONE eager launch with cudaProfilerStart/Stop (run under
`ncu --profile-from-start off`).  Prints one JSON line: us per launch, TFLOP/s, fraction of the
measured burst peak.
"""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2508_00960_b200.engine import PhantomEngine

KINDS = {"forward": ("ppx_forward_fused", "ppx_forward_n"), "error": ("ppx_error_phantoms_n", "ppx_error_phantoms",
         "ppx_error_phantoms_scatter"), "wgrad": ("ppx_wgrad",), "bwd": ("ppx_backward_fused",),
         "wgrad_errors": ("ppx_backward_wgrad_errors",),
         "recurrence": ("ppx_backward_delta_n",), "compress": ("ppx_compress_n",)}

ap = argparse.ArgumentParser()
ap.add_argument("kind", choices=sorted(KINDS))
ap.add_argument("--group", type=int, default=0)
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--index", type=int, default=-1, help="which matching launch of the step (default: middle)")
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--k3", default="auto", help="k3_fused plan: auto|0|1")
ap.add_argument("--noaccum", action="store_true", help="ppx_error_phantoms: overwrite instead of accumulate")
args = ap.parse_args()
if args.kind == "error" and not args.group:
    # the default one-GPU plan runs the error compression inside the first weight-gradient launch
    # of each layer (k3_grouped): probe the stand-alone launch of the alternative plan
    os.environ.setdefault("PPX_NO_K3G", "1")
cfg = bench.CONFIGS[args.config]
eng = PhantomEngine(cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"], lr=3e-6, group=args.group or None,
                    k3_fused=None if args.k3 == "auto" else args.k3 == "1")
xs, ts = bench.make_data(eng, 1, cfg)
for par in (0, 1):
    eng.set_batch(xs, ts, par)
eng.step(graph=False)
torch.cuda.synchronize()

# record the ABI calls of one eager step (arguments kept alive by the engine's _keep list)
calls = []
orig = eng.ctx.call


def rec(name, *a):
    calls.append((name, a))
    return orig(name, *a)


eng.ctx.call = rec
seq = eng.profile_step()
eng.ctx.call = orig
timed = {}
for nm, ms, fl in seq:
    timed.setdefault(nm, []).append((ms, fl))
match = [c for c in calls if c[0] in KINDS[args.kind]]
if not match:
    sys.exit(f"no {args.kind} launch in this plan: {sorted({c[0] for c in calls})}")
idx = len(match) // 2 if args.index < 0 else args.index
name, cargs = match[idx]
same = [c for c in match[:idx] if c[0] == name]          # ordinal of the pick among its ABI call
flops = [fl for nm, ms, fl in seq if nm == name][len(same)]
if args.noaccum and name == "ppx_error_phantoms":
    cargs = cargs[:6] + (0,) + cargs[7:]
keep = eng._keep            # the ctypes structs the recorded arguments point into
eng._keep = []              # never cleared again: the replays below reuse them


def launch():
    eng.ctx.call(name, *cargs)


S = torch.cuda.current_stream()
if args.ncu:
    launch()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    launch()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(json.dumps({"kind": args.kind, "call": name, "profiled": True}))
    sys.exit(0)
# the recorded stream handle is the eager step's stream (the current stream): replay on it
for _ in range(3):
    launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(200_000_000)
e0.record(S)
for _ in range(args.iters):
    launch()
e1.record(S)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / args.iters * 1e3
peak = bench.peaks()[0]
tf = flops / (us * 1e-6) / 1e12 if flops else None
print(json.dumps({"kind": args.kind, "call": name, "group": eng.group, "us_per_launch": us, "flops": flops,
                  "tflops": tf, "frac_of_burst": tf / peak if tf else None,
                  "step_profile_us": [round(ms * 1e3, 1) for ms, _ in timed.get(name, [])][:12]}))
