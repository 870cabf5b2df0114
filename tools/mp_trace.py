"""Per-ABI-call device time of one eager PhantomEngine step on N GPUs (torchrun), from CUDA events
recorded around every kernel launch (PhantomEngine.profile_step).  Rank 0 prints per-call totals and
the wall of the step.   torchrun --nproc-per-node N tools/mp_trace.py [--config c3]"""
import argparse, collections, json, os, sys
import torch
import torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_00960_b200 import _lib
from paper_2508_00960_b200.engine import PhantomEngine
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
uid = None
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    u = [_lib.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(u, src=0)
    uid = u[0]
eng = PhantomEngine(cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"], world=world, rank=rank, device=local,
                    uid=uid, lr=3e-6)
xs, ts = bench.make_data(eng, 1, cfg)
eng.set_batch(xs, ts, 0)
eng.set_batch(xs, ts, 1)
for _ in range(2):
    eng.step(graph=False)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
torch.cuda.synchronize()
S = torch.cuda.current_stream()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record(S)
seq = eng.profile_step()
t1.record(S)
torch.cuda.synchronize()
agg = collections.OrderedDict()
for name, ms, _fl in seq:
    x = agg.setdefault(name, [0, 0.0])
    x[0] += 1
    x[1] += ms * 1e3
out = {"rank": rank, "step_us": t0.elapsed_time(t1) * 1e3, "calls": {k: [v[0], round(v[1], 1)] for k, v in agg.items()},
       "seq": [(n, round(ms * 1e3, 1)) for n, ms, _f in seq]}
outs = [None] * world
if world > 1:
    dist.all_gather_object(outs, out)
else:
    outs = [out]
if rank == 0:
    for o in outs:
        print(f"rank {o['rank']}: eager step {o['step_us']:.0f} us")
        for k, (c, t) in o["calls"].items():
            print(f"   {k:24s} x{c:3d} {t:9.1f} us")
    json.dump(outs, open(os.path.join(ROOT, "gpurun_out", f"mp_trace_{args.config}_n{world}.json"), "w"))
if world > 1:
    dist.barrier()
eng.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
