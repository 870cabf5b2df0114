"""Measure NCCL collectives over NVLink 5 / NVSwitch on this box and fit the paper's comm model
(reference collectives.py:471-535): time_us = c1*log2(p) + c2*m + c3.

    torchrun --nproc-per-node 4 tools/comm_fit.py --out profiles/comm_b200
writes <out>.csv (collective,m,p,time_us; m = bf16 elements per rank) and <out>.ini.
Every group size 2..world (the first p ranks) is measured; times are CUDA-event medians on each
rank, max over ranks.
"""
import argparse
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/comm_b200")
    ap.add_argument("--max-log2", type=int, default=26)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    from paper_2508_00960_b200.collectives import Collective
    from paper_2508_00960_b200.commmodel import fit_comm_model, save_comm_model, save_measurements
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    samples = []
    for p in range(2, world + 1):
        group = dist.new_group(list(range(p)))
        for lg in range(2, a.max_log2 + 1, 2):
            m = 1 << lg
            if rank < p:
                x = torch.randn(m, device="cuda").to(torch.bfloat16)
                big = torch.empty(p * m, dtype=torch.bfloat16, device="cuda")
                ops = {
                    Collective.ALL_GATHER: lambda: dist.all_gather_into_tensor(big, x, group=group),
                    Collective.REDUCE_SCATTER: lambda: dist.reduce_scatter_tensor(x, big, group=group),
                    Collective.ALL_REDUCE: lambda: dist.all_reduce(x, group=group),
                    Collective.BROADCAST: lambda: dist.broadcast(x, src=0, group=group),
                }
                for kind, op in ops.items():
                    for _ in range(5):
                        op()
                    ts = []
                    for _ in range(a.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        dist.barrier(group=group)
                        e0.record()
                        op()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e3)
                    t = torch.tensor([statistics.median(ts)], device="cuda")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                    samples.append((kind, m, p, float(t.item())))
            dist.barrier()
    if rank == 0:
        save_measurements(samples, a.out + ".csv")
        model = fit_comm_model(samples)
        save_comm_model(model, a.out + ".ini")
        for kind, c in model.costs.items():
            print(f"{kind.value:15s} c1={c.c1:.3f} us/log2p  c2={c.c2 * 1e6:.4f} us/Melem  c3={c.c3:.2f} us  "
                  f"rmse={2 ** model.rmse_log2_us[kind]:.2f} us")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
