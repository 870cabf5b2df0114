"""Multi-GPU parity of the tensor-parallel comparison pipeline: TPEngine (Megatron column/row
pairs, NCCL all-reduces) on N GPUs (torchrun, one process per GPU) vs the dense float64 oracle —
TP is an exact reparameterisation of the dense FFN (reference tensor_parallel.py:67-153,
training.py:216-244; test_acceptance.py:100-118).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mp_tp_parity.py [--dtype fp32|bf16]

Compares every step's loss and each GPU's weight UPDATES (its row block of the column-parallel
layers, its column block of the row-parallel layers, both biases) with the oracle's.
Tolerances: fp32 tier 1e-4 losses and updates — an update is measured from the engine's own
fp32 master after loading, and its tolerance is raised to the fp32 master's representation floor
4 * 2^-24 * ||W|| / ||dW|| where that is larger (a fp32 weight cannot carry a smaller update more
precisely); bf16 tier 2e-2 losses, 1e-1 updates.  Rank 0 prints one JSON verdict.
"""
import argparse, json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phantom_oracle as po
from paper_2508_00960_b200 import _lib
from paper_2508_00960_b200.tensor_parallel import TPEngine


def nerr(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--lr", type=float, default=3e-3)
    ap.add_argument("--graph", type=int, default=1)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [_lib.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    n, L, B, lr = args.width, args.layers, args.B, args.lr
    f32 = args.dtype == "fp32"
    dtype = torch.float32 if f32 else torch.bfloat16
    tol_l, tol_u = (1e-4, 1e-4) if f32 else (2e-2, 1e-1)
    rng = np.random.default_rng(5)
    a = np.sqrt(6.0 / (2 * n))
    W = [rng.uniform(-a, a, (n, n)) for _ in range(L)]
    b = [0.1 * rng.standard_normal(n) for _ in range(L)]
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = TPEngine(n, L, B, world=world, rank=rank, device=local, uid=uid[0], lr=lr, dtype=dtype)
    eng.load_full_weights(W, b)
    s = n // world
    r0, r1 = rank * s, (rank + 1) * s
    start = [t.double().cpu().numpy().copy() for m in range(L // 2)
             for t in (eng.Wa[m], eng.Wb[m], eng._ba(m), eng._bb(m))]
    for par in (0, 1):
        eng.set_batch(torch.from_numpy(x.T.copy()).cuda(), torch.from_numpy(y.T.copy()).cuda(), par)
    losses = []
    eng.step(graph=False)
    losses.append(eng.read_loss())
    if args.steps > 1 and args.graph:
        eng.capture()
    for _ in range(args.steps - 1):
        eng.step(graph=bool(args.graph))
        losses.append(eng.read_loss())
    Wd = [w.copy() for w in W]
    bd = [v.copy() for v in b]
    ref = []
    for _ in range(args.steps):
        out = po.tp_iteration([[{"weight": Wd[l], "bias": bd[l]} for l in range(L)]], ["relu"] * L, [x], [y], "mean")
        ref.append(out["global_loss"])
        for l in range(L):
            Wd[l] -= lr * out["grads"][0][l]["weight"]
            bd[l] -= lr * out["grads"][0][l]["bias"]
    worst = {"loss": max(abs(g - r) / abs(r) for g, r in zip(losses, ref)), "update_over_tol": 0.0,
             "update": 0.0}
    i = 0
    per = {}
    for m in range(L // 2):
        upd = [(eng.Wa[m], W[2 * m][r0:r1, :], Wd[2 * m][r0:r1, :]),
               (eng.Wb[m], W[2 * m + 1][:, r0:r1], Wd[2 * m + 1][:, r0:r1]),
               (eng._ba(m), b[2 * m][r0:r1], bd[2 * m][r0:r1]),
               (eng._bb(m), b[2 * m + 1], bd[2 * m + 1])]
        for got, w0, w1 in upd:
            want = w1 - w0
            e = nerr(got.double().cpu().numpy() - start[i], want)
            floor = 4 * 2.0 ** -24 * np.linalg.norm(w1) / max(np.linalg.norm(want), 1e-300) if f32 else 0.0
            worst["update"] = max(worst["update"], e)
            worst["update_over_tol"] = max(worst["update_over_tol"], e / max(tol_u, floor))
            per[f"{('Wa', 'Wb', 'ba', 'bb')[i % 4]}{m}"] = (round(e, 7), round(floor, 7))
            i += 1
    w = torch.tensor([worst["loss"], worst["update_over_tol"], worst["update"]], device="cuda", dtype=torch.float64)
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    ok = bool(w[0] <= tol_l and w[1] <= 1.0)
    if rank == 0:
        print(json.dumps({"world": world, "dtype": args.dtype, "losses": losses, "oracle": ref,
                          "worst": {"loss": float(w[0]), "update": float(w[2]), "update_over_tol": float(w[1])},
                          "tol": {"loss": tol_l, "update": tol_u}, "rank0_per_tensor_err_floor": per, "pass": ok}), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    sys.exit(main())
