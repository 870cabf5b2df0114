"""Graph-replayed step time of the default plan (torchrun for N > 1), for same-box A/B of planner
or debug switches that bench.py refuses:  torchrun --nproc-per-node N tools/step_time.py [--config c3]"""
import argparse, json, os, sys
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2508_00960_b200.engine import PhantomEngine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--group", type=int, default=0, help="logical ranks per launch (1 = the 8-GPU per-GPU shapes)")
ap.add_argument("--k3", default="auto", choices=["auto", "0", "1"], help="k3_fused plan A/B")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
world, rank, local = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
D = bench.Dist(world, rank, local)
eng = PhantomEngine(cfg["n"], cfg["p"], cfg["k"], cfg["layers"], cfg["batch"], world=world, rank=rank, device=local,
                    uid=D.uid(), lr=3e-6, group=a.group or None,
                    k3_fused=None if a.k3 == "auto" else a.k3 == "1")
xs, ts = bench.make_data(eng, 1234, cfg)
eng.set_batch(xs, ts, 0)
eng.set_batch(xs, ts, 1)
eng.step(graph=False)
eng.capture()
for _ in range(5):
    eng.step()
ms = [bench.timed_steps(eng, D, a.steps) for _ in range(a.reps)]
if rank == 0:
    env = {k: v for k, v in os.environ.items() if k.startswith(("PPX_DEBUG", "PPX_NO_", "PPX_AB_"))}
    print(json.dumps({"config": a.config, "world": world, "group": eng.group, "k3": eng.k3_fused, "env": env, "ms": ms}))
D.barrier()
eng.close()
bench.finish(D)
