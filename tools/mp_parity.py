"""Multi-GPU parity: PhantomEngine over NCCL (torchrun, one process per GPU) vs the CPU oracle.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mp_parity.py [--dtype fp32|bf16]
Each process owns p/N logical ranks; after `steps` SGD steps every process compares its shards'
weights and the global loss with oracle/phantom_oracle.py and rank 0 prints one JSON verdict.
"""
import argparse, json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import phantom_oracle as po
from paper_2508_00960_b200 import _lib
from paper_2508_00960_b200.engine import PhantomEngine


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--lr", type=float, default=3e-3)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [_lib.Context.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    n, p, k, L, B, lr = args.width, args.p, args.k, 3, args.B, args.lr
    dtype = torch.float32 if args.dtype == "fp32" else torch.bfloat16
    tol = 1e-4 if args.dtype == "fp32" else 2e-2
    model = po.init_phantom_model(n, p, k, L, 3)
    rng = np.random.default_rng(3)
    for row in model:
        for lay in row:
            lay["bias"] = 0.1 * rng.standard_normal(lay["bias"].shape)
    x = rng.standard_normal((n, B))
    y = np.maximum(rng.standard_normal((n, B)), 0.0)
    eng = PhantomEngine(n, p, k, L, B, world=world, rank=rank, device=local, uid=uid[0], lr=lr, dtype=dtype)
    eng.load_params(model)
    s = n // p
    xs = [torch.from_numpy(x[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local]
    ys = [torch.from_numpy(y[j * s:(j + 1) * s].T.copy()).cuda() for j in eng.local]
    eng.set_batch(xs, ys, 0)
    eng.set_batch(xs, ys, 1)
    if args.graph:
        eng.capture()
    losses = []
    for _ in range(args.steps):
        eng.step(graph=bool(args.graph))
        losses.append(eng.read_loss())
    ref = []
    for _ in range(args.steps):
        out = po.pp_iteration(model, ["relu"] * L, [x[j * s:(j + 1) * s] for j in range(p)],
                              [y[j * s:(j + 1) * s] for j in range(p)], "mean")
        ref.append(out["global_loss"])
        for j in range(p):
            params, gs = po.pp_param_list(model[j], out["grads"][j])
            po.sgd_step(params, gs, lr)
    worst = max(abs(a - b) / abs(b) for a, b in zip(losses, ref))
    for jj, j in enumerate(eng.local):
        for l in range(L):
            v = eng.layer_views(jj, l)
            for name in ("local", "compressor", "bias"):
                a = v[name].double().cpu().numpy()
                b = model[j][l][name]
                worst = max(worst, np.linalg.norm(a - b) / np.linalg.norm(b))
            for i, d in v["decompressors"].items():
                b = model[j][l]["decompressors"][i]
                worst = max(worst, np.linalg.norm(d.double().cpu().numpy() - b) / np.linalg.norm(b))
    w = torch.tensor([worst], device="cuda")
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"world": world, "dtype": args.dtype, "graph": args.graph, "losses": losses, "oracle": ref,
                          "worst_rel_err": float(w.item()), "tol": tol, "fused": bool(eng.fused), "p2p": eng.p2p, "pass": float(w.item()) <= tol}), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    print('[teardown] closing engine', file=sys.stderr, flush=True)
    eng.close()
    print('[teardown] engine closed', file=sys.stderr, flush=True)
    dist.barrier()
    dist.destroy_process_group()
    print('[teardown] pg destroyed', file=sys.stderr, flush=True)
    sys.stdout.flush()
    os._exit(0 if float(w.item()) <= tol else 1)


if __name__ == "__main__":
    sys.exit(main())
