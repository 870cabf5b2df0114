"""Fixed-loss PP-vs-TP comparison on B200 (reference cli.py:335-402 `compare`,
test_acceptance.py:226-250): train the same-width Megatron TP FFN for E epochs, set the target to
1.05x its final epoch loss, train the phantom model until it reaches that target, and report
epochs, seconds and measured NVML joules to target for both (one JSON line on rank 0).

    python tools/compare_pp_tp.py [--n 8192 --p 8 --k 64 --layers 4 ...]
    torchrun --nproc-per-node N tools/compare_pp_tp.py ...   (N GPUs; p logical ranks over them)
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--samples", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--lr", type=float, default=3e-6)   # 1e-5 diverges (non-finite) for the PP model at n=8192
    ap.add_argument("--tp-epochs", type=int, default=20)
    ap.add_argument("--max-epochs", type=int, default=200)
    ap.add_argument("--slack", type=float, default=1.05)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2508_00960_b200 import _lib
    from paper_2508_00960_b200.training import TrainConfig, gen_dataset_device, train_engine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def new_uid():
        u = [_lib.Context.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(u, src=0)
        return u[0]

    data = gen_dataset_device(a.n, a.samples, seed=0)
    common = dict(n=a.n, layers=a.layers, batch=a.batch, lr=a.lr, seed=0, loss_reduction="mean",
                  dtype=torch.bfloat16)
    tp_cfg = TrainConfig(mode="tp", p=world, max_epochs=a.tp_epochs, **common)
    tp = train_engine(tp_cfg, data, world=world, rank=rank, device=local, uid=new_uid() if world > 1 else None)
    target = a.slack * tp.loss_history[-1]
    pp_cfg = TrainConfig(mode="pp", p=a.p, k=a.k, max_epochs=a.max_epochs, target_loss=target, optimizer="sgd",
                         **common)
    from paper_2508_00960_b200.errors import TrainingError
    try:
        pp = train_engine(pp_cfg, data, world=world, rank=rank, device=local, uid=new_uid() if world > 1 else None,
                          init="device")
    except TrainingError as exc:   # the phantom model diverged at this learning rate: say so
        if rank == 0:
            line = {"config": {"n": a.n, "p_pp": a.p, "k": a.k, "layers": a.layers, "lr": a.lr, "gpus": world},
                    "target_loss": target, "tp_loss_history": tp.loss_history, "pp_diverged": str(exc)}
            print(json.dumps(line))
            if a.out:
                json.dump(line, open(a.out, "w"), indent=1)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    def joules(r):
        j = torch.tensor([r.cost["joules"] if r.cost["joules"] is not None else float("nan")], device="cuda")
        if world > 1:
            dist.all_reduce(j)
        return float(j.item())

    tpj, ppj = joules(tp), joules(pp)
    # TP time / energy to its own first epoch at or below the target
    tp_hit = next((e + 1 for e, v in enumerate(tp.loss_history) if v <= target), tp.epochs_run)
    frac = tp_hit / max(1, tp.epochs_run)
    line = {
        "config": {"n": a.n, "p_pp": a.p, "k": a.k, "layers": a.layers, "samples": a.samples, "batch": a.batch,
                   "lr": a.lr, "gpus": world, "dtype": "bf16", "data": "synthetic teacher (device RNG)"},
        "target_loss": target,
        "tp": {"epochs_run": tp.epochs_run, "epochs_to_target": tp_hit, "seconds": tp.cost["seconds"],
               "seconds_to_target": tp.cost["seconds"] * frac, "joules_to_target": tpj * frac,
               "j_per_epoch": tpj / max(1, tp.epochs_run), "samples_per_s": tp.cost["samples_per_s"],
               "loss_history": tp.loss_history},
        "pp": {"epochs_to_target": pp.epochs_run, "converged": pp.converged, "seconds_to_target": pp.cost["seconds"],
               "joules_to_target": ppj, "j_per_epoch": ppj / max(1, pp.epochs_run),
               "samples_per_s": pp.cost["samples_per_s"], "loss_history": pp.loss_history},
    }
    if pp.converged:
        line["energy_ratio_pp_over_tp"] = ppj / (tpj * frac) if tpj == tpj and tpj > 0 else None
        line["time_ratio_pp_over_tp"] = pp.cost["seconds"] / (tp.cost["seconds"] * frac)
    if rank == 0:
        print(json.dumps(line))
        if a.out:
            with open(a.out, "w") as fh:
                json.dump(line, fh, indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
